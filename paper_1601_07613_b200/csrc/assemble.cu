// Surface extraction on the GPU: the reference's
// mesh.assemble (/root/reference/pkg/src/meshchroma/mesh.py:207-300)
// restated as sort + scan, bit-identical ids:
//   * every element side becomes one slot (element-major, side-minor);
//     its sorted vertex tuple is packed into one 64-bit key;
//   * a stable radix sort (CUB) groups equal keys with slots ascending;
//   * surfaces are numbered by first encounter: the id of a group is the
//     number of group-first slots that precede its first slot in slot order
//     (an exclusive scan over a slot-indexed mark array, no second sort);
//   * left = element of the first slot (the smaller id), right = element
//     of the second slot, -1 for boundary surfaces; > 2 slots = non-manifold.
// The reference uses np.unique(axis=0) (~63 s of c4 generation).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "mc_internal.h"

namespace {

constexpr unsigned long long kInvalid = ~0ull;

// local side tables (mesh.py:51-55): tri, quad, tet; -1 padded
__constant__ int c_sides[3][4][3] = {
    {{0, 1, -1}, {1, 2, -1}, {2, 0, -1}, {-1, -1, -1}},
    {{0, 1, -1}, {1, 2, -1}, {2, 3, -1}, {3, 0, -1}},
    {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}}};

__global__ void k_keys(const int64_t* __restrict__ ev, const int8_t* __restrict__ kind,
                       int64_t ne, int width, uint64_t nv, unsigned long long* keys,
                       int64_t* slots) {
  const int64_t n = ne * 4;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = t >> 2;
    const int side = int(t & 3);
    const int k = kind[e];
    unsigned long long key = kInvalid;
    if (c_sides[k][side][0] >= 0) {
      uint64_t v[3];
      const int w = c_sides[k][side][2] >= 0 ? 3 : 2;
      for (int i = 0; i < w; ++i) v[i] = uint64_t(ev[e * 4 + c_sides[k][side][i]]);
      // sort the tuple
      if (v[0] > v[1]) { uint64_t x = v[0]; v[0] = v[1]; v[1] = x; }
      if (w == 3) {
        if (v[1] > v[2]) { uint64_t x = v[1]; v[1] = v[2]; v[2] = x; }
        if (v[0] > v[1]) { uint64_t x = v[0]; v[0] = v[1]; v[1] = x; }
        key = (v[0] * nv + v[1]) * nv + v[2];
      } else {
        key = v[0] * nv + v[1];
      }
      (void)width;
    }
    keys[t] = key;
    slots[t] = t;
  }
}

// heads of equal-key runs in sorted order; mark[first slot] = 1
__global__ void k_heads(const unsigned long long* __restrict__ sk, const int64_t* __restrict__ ss,
                        int64_t n, int32_t* head, int32_t* mark) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const bool h = sk[i] != kInvalid && (i == 0 || sk[i] != sk[i - 1]);
    head[i] = h ? 1 : 0;
    if (h) mark[ss[i]] = 1;
  }
}

// per sorted position: surface id of its group = rank of the group's first
// slot among first slots (exclusive scan of mark, indexed by slot)
__global__ void k_assign(const unsigned long long* __restrict__ sk, const int64_t* __restrict__ ss,
                         const int32_t* __restrict__ head_scan, const int32_t* __restrict__ head,
                         const int32_t* __restrict__ mark_scan, int64_t n, int64_t* group_first,
                         int32_t* group_count, int64_t* elem_surfs) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (sk[i] == kInvalid) {
      elem_surfs[ss[i]] = -1;
      continue;
    }
    const int32_t g = head_scan[i] + head[i] - 1;   // inclusive group index
    if (head[i]) group_first[g] = i;
    atomicAdd(&group_count[g], 1);
    (void)mark_scan;
  }
}

__global__ void k_outputs(const unsigned long long* __restrict__ sk, const int64_t* __restrict__ ss,
                          const int64_t* __restrict__ group_first,
                          const int32_t* __restrict__ group_count,
                          const int32_t* __restrict__ mark_scan, const int64_t* __restrict__ ev,
                          const int8_t* __restrict__ kind, int64_t ngroups, int width,
                          int64_t* surf_verts, int64_t* surf_elems, int64_t* elem_surfs,
                          int32_t* surf_count, unsigned long long* bad) {
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < ngroups;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i0 = group_first[g];
    const int64_t slot0 = ss[i0];
    const int64_t sid = mark_scan[slot0];           // first-encounter id
    const int cnt = group_count[g];
    for (int c = 0; c < cnt; ++c) elem_surfs[ss[i0 + c]] = sid;
    surf_count[sid] = cnt;
    surf_elems[2 * sid] = slot0 >> 2;
    surf_elems[2 * sid + 1] = cnt >= 2 ? (ss[i0 + 1] >> 2) : -1;
    if (cnt > 2) atomicMin(bad, static_cast<unsigned long long>(sid));
    // sorted vertex tuple of the first slot
    const int64_t e = slot0 >> 2;
    const int side = int(slot0 & 3);
    const int k = kind[e];
    int64_t v[3];
    for (int q = 0; q < width; ++q) v[q] = ev[e * 4 + c_sides[k][side][q]];
    if (v[0] > v[1]) { int64_t x = v[0]; v[0] = v[1]; v[1] = x; }
    if (width == 3) {
      if (v[1] > v[2]) { int64_t x = v[1]; v[1] = v[2]; v[2] = x; }
      if (v[0] > v[1]) { int64_t x = v[0]; v[0] = v[1]; v[1] = x; }
    }
    for (int q = 0; q < width; ++q) surf_verts[sid * width + q] = v[q];
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return int(g < 1 ? 1 : g);
}

}  // namespace

struct mc_assembly {
  int64_t ne = 0, ns = 0;
  int width = 2;
  int64_t *d_surf_verts = nullptr, *d_surf_elems = nullptr, *d_elem_surfs = nullptr;
  int32_t* d_surf_count = nullptr;
  int64_t bad_sid = -1;
};

#define AS_TRY(expr)                                                                    \
  do {                                                                                  \
    cudaError_t e__ = (expr);                                                           \
    if (e__ != cudaSuccess) {                                                           \
      rc = mc_fail(MC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));      \
      goto done;                                                                        \
    }                                                                                   \
  } while (0)

extern "C" {

MC_API int mc_assemble_create(int64_t n_elements, int64_t n_vertices, const int8_t* kind_codes,
                              const int64_t* elem_verts, int width, mc_assembly** out,
                              int64_t* n_surfaces) {
  if (!out || !n_surfaces || !kind_codes || !elem_verts) return mc_fail(MC_EINVAL, "null argument");
  *out = nullptr;
  if (n_elements <= 0 || (width != 2 && width != 3)) return mc_fail(MC_EINVAL, "bad sizes");
  const double kmax = width == 2 ? double(n_vertices) * n_vertices
                                 : double(n_vertices) * n_vertices * n_vertices;
  if (kmax >= 1.8e19)
    return mc_fail(MC_EUNSUPPORTED, "vertex count too large for 64-bit side keys");
  for (int64_t e = 0; e < n_elements; ++e)
    if (kind_codes[e] < 0 || kind_codes[e] > 2) return mc_fail(MC_EINVAL, "bad element kind");
  const int64_t n = n_elements * 4;
  int rc = MC_OK;
  int64_t *d_ev = nullptr, *d_slots = nullptr, *d_slots2 = nullptr, *d_first = nullptr;
  int8_t* d_kind = nullptr;
  unsigned long long *d_keys = nullptr, *d_keys2 = nullptr, *d_bad = nullptr;
  int32_t *d_head = nullptr, *d_hscan = nullptr, *d_mark = nullptr, *d_mscan = nullptr,
          *d_count = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0, t1 = 0, t2 = 0, t3 = 0;
  int32_t ngroups_last[2] = {0, 0};
  int64_t ngroups = 0;
  unsigned long long bad = ~0ull;
  auto A = new mc_assembly();
  A->ne = n_elements;
  A->width = width;
  int end_bit = 64;
  {
    // only the bits the keys can use
    const double km = kmax < 1 ? 1 : kmax;
    int b = 1;
    while (b < 64 && double(1ull << b) <= km) ++b;
    end_bit = b;
  }
  AS_TRY(cudaMalloc(&d_ev, sizeof(int64_t) * n));
  AS_TRY(cudaMalloc(&d_kind, n_elements));
  AS_TRY(cudaMalloc(&d_keys, sizeof(unsigned long long) * n));
  AS_TRY(cudaMalloc(&d_keys2, sizeof(unsigned long long) * n));
  AS_TRY(cudaMalloc(&d_slots, sizeof(int64_t) * n));
  AS_TRY(cudaMalloc(&d_slots2, sizeof(int64_t) * n));
  AS_TRY(cudaMalloc(&d_head, sizeof(int32_t) * n));
  AS_TRY(cudaMalloc(&d_hscan, sizeof(int32_t) * n));
  AS_TRY(cudaMalloc(&d_mark, sizeof(int32_t) * n));
  AS_TRY(cudaMalloc(&d_mscan, sizeof(int32_t) * n));
  AS_TRY(cudaMalloc(&d_bad, sizeof(unsigned long long)));
  AS_TRY(cudaMemcpy(d_ev, elem_verts, sizeof(int64_t) * n, cudaMemcpyHostToDevice));
  AS_TRY(cudaMemcpy(d_kind, kind_codes, n_elements, cudaMemcpyHostToDevice));
  AS_TRY(cudaMemset(d_mark, 0, sizeof(int32_t) * n));
  AS_TRY(cudaMemcpy(d_bad, &bad, sizeof(bad), cudaMemcpyHostToDevice));
  k_keys<<<grid_for(n), 256>>>(d_ev, d_kind, n_elements, width, uint64_t(n_vertices), d_keys,
                               d_slots);
  AS_TRY(cudaGetLastError());
  // stable sort: invalid keys (all ones) land at the end; restrict radix bits
  // to the used range plus the all-ones pattern
  AS_TRY(cub::DeviceRadixSort::SortPairs(nullptr, t1, d_keys, d_keys2, d_slots, d_slots2, n, 0, 64));
  AS_TRY(cub::DeviceScan::ExclusiveSum(nullptr, t2, d_head, d_hscan, n));
  tmp_bytes = t1 > t2 ? t1 : t2;
  AS_TRY(cudaMalloc(&d_tmp, tmp_bytes));
  (void)t3;
  (void)end_bit;
  AS_TRY(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_keys, d_keys2, d_slots, d_slots2, n,
                                         0, 64));
  k_heads<<<grid_for(n), 256>>>(d_keys2, d_slots2, n, d_head, d_mark);
  AS_TRY(cudaGetLastError());
  AS_TRY(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_head, d_hscan, n));
  AS_TRY(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_mark, d_mscan, n));
  AS_TRY(cudaMemcpy(&ngroups_last[0], d_hscan + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost));
  AS_TRY(cudaMemcpy(&ngroups_last[1], d_head + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost));
  ngroups = int64_t(ngroups_last[0]) + ngroups_last[1];
  A->ns = ngroups;
  AS_TRY(cudaMalloc(&d_first, sizeof(int64_t) * (ngroups + 1)));
  AS_TRY(cudaMalloc(&d_count, sizeof(int32_t) * (ngroups + 1)));
  AS_TRY(cudaMemset(d_count, 0, sizeof(int32_t) * (ngroups + 1)));
  AS_TRY(cudaMalloc(&A->d_surf_verts, sizeof(int64_t) * (ngroups * width + 1)));
  AS_TRY(cudaMalloc(&A->d_surf_elems, sizeof(int64_t) * (ngroups * 2 + 1)));
  AS_TRY(cudaMalloc(&A->d_elem_surfs, sizeof(int64_t) * n));
  AS_TRY(cudaMalloc(&A->d_surf_count, sizeof(int32_t) * (ngroups + 1)));
  k_assign<<<grid_for(n), 256>>>(d_keys2, d_slots2, d_hscan, d_head, d_mscan, n, d_first, d_count,
                                 A->d_elem_surfs);
  AS_TRY(cudaGetLastError());
  k_outputs<<<grid_for(ngroups), 256>>>(d_keys2, d_slots2, d_first, d_count, d_mscan, d_ev, d_kind,
                                        ngroups, width, A->d_surf_verts, A->d_surf_elems,
                                        A->d_elem_surfs, A->d_surf_count, d_bad);
  AS_TRY(cudaGetLastError());
  AS_TRY(cudaMemcpy(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost));
  A->bad_sid = bad == ~0ull ? -1 : int64_t(bad);
done:
  cudaFree(d_ev);
  cudaFree(d_kind);
  cudaFree(d_keys);
  cudaFree(d_keys2);
  cudaFree(d_slots);
  cudaFree(d_slots2);
  cudaFree(d_head);
  cudaFree(d_hscan);
  cudaFree(d_mark);
  cudaFree(d_mscan);
  cudaFree(d_first);
  cudaFree(d_count);
  cudaFree(d_bad);
  cudaFree(d_tmp);
  if (rc != MC_OK) {
    mc_assemble_destroy(A);
    return rc;
  }
  *out = A;
  *n_surfaces = A->ns;
  if (A->bad_sid >= 0) {
    mc_set_error("surface " + std::to_string(A->bad_sid) + " is shared by more than two elements");
    return MC_ENONMANIFOLD;
  }
  return MC_OK;
}

MC_API int mc_assemble_result(mc_assembly* A, int64_t* surf_verts, int64_t* surf_elems,
                              int64_t* elem_surfs, int32_t* surf_count) {
  if (!A) return mc_fail(MC_EINVAL, "null handle");
  cudaError_t e = cudaSuccess;
  if (surf_verts)
    e = cudaMemcpy(surf_verts, A->d_surf_verts, sizeof(int64_t) * A->ns * A->width,
                   cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && surf_elems)
    e = cudaMemcpy(surf_elems, A->d_surf_elems, sizeof(int64_t) * A->ns * 2, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && elem_surfs)
    e = cudaMemcpy(elem_surfs, A->d_elem_surfs, sizeof(int64_t) * A->ne * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && surf_count)
    e = cudaMemcpy(surf_count, A->d_surf_count, sizeof(int32_t) * A->ns, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mc_fail(MC_ECUDA, std::string("assembly download: ") + cudaGetErrorString(e));
  return MC_OK;
}

MC_API int mc_assemble_destroy(mc_assembly* A) {
  if (!A) return MC_OK;
  cudaFree(A->d_surf_verts);
  cudaFree(A->d_surf_elems);
  cudaFree(A->d_elem_surfs);
  cudaFree(A->d_surf_count);
  delete A;
  return MC_OK;
}

}  // extern "C"
