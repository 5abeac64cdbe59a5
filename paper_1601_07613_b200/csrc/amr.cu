// AMR split-edge color propagation on the GPU: the
// per-fine-surface classification and coloring of the reference's
// _materialize (/root/reference/pkg/src/meshchroma/amr.py:221-245, colors
// :158-164, child_color :52-58, parallel rule :47,263), one thread per fine
// surface.  Base edges are found by binary search over the base edge keys
// sorted on the device (CUB radix sort), never by a host dictionary.
//
//   origin 0  whole base edge        -> color of that edge
//   origin 1  half of a split edge   -> (c + 3m - 4) % 6 + 1, m = 1 for the
//                                       half holding the lower base vertex
//   origin 2  interior child edge    -> color of the parent edge joining the
//                                       two far endpoints (parallel edge)
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "mc_internal.h"

namespace {

__device__ __forceinline__ int64_t find_base(const unsigned long long* keys,
                                             const int64_t* sids, int64_t n,
                                             unsigned long long k) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && keys[lo] == k) ? sids[lo] : -1;
}

__device__ __forceinline__ unsigned long long edge_key(int64_t u, int64_t w, int64_t nv) {
  const int64_t a = u < w ? u : w, b = u < w ? w : u;
  return static_cast<unsigned long long>(a) * static_cast<unsigned long long>(nv) +
         static_cast<unsigned long long>(b);
}

__global__ void k_base_keys(const int64_t* __restrict__ bsv, int64_t nbs, int64_t nv,
                            unsigned long long* keys, int64_t* sids) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < nbs;
       s += int64_t(gridDim.x) * blockDim.x) {
    keys[s] = edge_key(bsv[2 * s], bsv[2 * s + 1], nv);
    sids[s] = s;
  }
}

__global__ void k_classify(const int64_t* __restrict__ fsv, int64_t ns, int64_t nbv,
                           const int64_t* __restrict__ split, const int64_t* __restrict__ bsv,
                           const int32_t* __restrict__ bcol, const unsigned long long* keys,
                           const int64_t* sids, int64_t nbs, int8_t* origin, int64_t* base_surface,
                           int8_t* half_index, int32_t* colors, int* err) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < ns;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t a = fsv[2 * s], b = fsv[2 * s + 1];   // sorted: a < b
    int8_t o, h = 0;
    int64_t bs;
    int32_t c;
    if (b < nbv) {                       // whole base edge
      o = 0;
      bs = find_base(keys, sids, nbs, edge_key(a, b, nbv));
      if (bs < 0) { atomicExch(err, 1); bs = 0; }
      c = bcol[bs];
    } else if (a < nbv) {                // half: a base vertex and a midpoint
      o = 1;
      bs = split[b - nbv];
      h = (a == bsv[2 * bs]) ? 1 : 2;
      c = (bcol[bs] + 3 * h - 4) % 6 + 1;
    } else {                             // interior edge between two midpoints
      o = 2;
      const int64_t* e1 = bsv + 2 * split[a - nbv];
      const int64_t* e2 = bsv + 2 * split[b - nbv];
      const bool c00 = e1[0] == e2[0], c01 = e1[0] == e2[1];
      const bool c10 = e1[1] == e2[0], c11 = e1[1] == e2[1];
      if (int(c00) + int(c01) + int(c10) + int(c11) != 1) atomicExch(err, 2);
      const int64_t common = (c00 || c01) ? e1[0] : e1[1];
      const int64_t x = e1[0] + e1[1] - common, y = e2[0] + e2[1] - common;
      bs = find_base(keys, sids, nbs, edge_key(x, y, nbv));
      if (bs < 0) { atomicExch(err, 1); bs = 0; }
      c = bcol[bs];
    }
    origin[s] = o;
    base_surface[s] = bs;
    half_index[s] = h;
    colors[s] = c;
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return int(g < 1 ? 1 : g);
}

}  // namespace

#define AMR_TRY(expr)                                                                   \
  do {                                                                                  \
    cudaError_t e__ = (expr);                                                           \
    if (e__ != cudaSuccess) {                                                           \
      rc = mc_fail(MC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));      \
      goto done;                                                                        \
    }                                                                                   \
  } while (0)

extern "C" {

MC_API int mc_amr_classify(int64_t n_fine_surfaces, const int64_t* fine_surf_verts,
                           int64_t n_base_vertices, int64_t n_split, const int64_t* split,
                           int64_t n_base_surfaces, const int64_t* base_surf_verts,
                           const int32_t* base_colors, int8_t* surf_origin,
                           int64_t* base_surface, int8_t* half_index, int32_t* colors) {
  if (n_fine_surfaces < 0 || n_base_surfaces <= 0 || n_split < 0 || !fine_surf_verts ||
      !base_surf_verts || !base_colors || !surf_origin || !base_surface || !half_index ||
      !colors || (n_split > 0 && !split))
    return mc_fail(MC_EINVAL, "bad arguments");
  if (double(n_base_vertices) * double(n_base_vertices) >= 1.8e19)
    return mc_fail(MC_EUNSUPPORTED, "vertex count too large for 64-bit edge keys");
  const int64_t ns = n_fine_surfaces, nbs = n_base_surfaces;
  int rc = MC_OK;
  int64_t *d_fsv = nullptr, *d_split = nullptr, *d_bsv = nullptr, *d_sid = nullptr,
          *d_sid2 = nullptr, *d_bs = nullptr;
  unsigned long long *d_key = nullptr, *d_key2 = nullptr;
  int32_t *d_bcol = nullptr, *d_col = nullptr;
  int8_t *d_org = nullptr, *d_half = nullptr;
  int* d_err = nullptr;
  void* d_tmp = nullptr;
  size_t tmp = 0;
  int herr = 0;
  AMR_TRY(cudaMalloc(&d_fsv, sizeof(int64_t) * (2 * ns + 1)));
  AMR_TRY(cudaMalloc(&d_split, sizeof(int64_t) * (n_split + 1)));
  AMR_TRY(cudaMalloc(&d_bsv, sizeof(int64_t) * 2 * nbs));
  AMR_TRY(cudaMalloc(&d_sid, sizeof(int64_t) * nbs));
  AMR_TRY(cudaMalloc(&d_sid2, sizeof(int64_t) * nbs));
  AMR_TRY(cudaMalloc(&d_key, sizeof(unsigned long long) * nbs));
  AMR_TRY(cudaMalloc(&d_key2, sizeof(unsigned long long) * nbs));
  AMR_TRY(cudaMalloc(&d_bcol, sizeof(int32_t) * nbs));
  AMR_TRY(cudaMalloc(&d_bs, sizeof(int64_t) * (ns + 1)));
  AMR_TRY(cudaMalloc(&d_col, sizeof(int32_t) * (ns + 1)));
  AMR_TRY(cudaMalloc(&d_org, ns + 1));
  AMR_TRY(cudaMalloc(&d_half, ns + 1));
  AMR_TRY(cudaMalloc(&d_err, sizeof(int)));
  AMR_TRY(cudaMemset(d_err, 0, sizeof(int)));
  if (ns) AMR_TRY(cudaMemcpy(d_fsv, fine_surf_verts, sizeof(int64_t) * 2 * ns, cudaMemcpyHostToDevice));
  if (n_split) AMR_TRY(cudaMemcpy(d_split, split, sizeof(int64_t) * n_split, cudaMemcpyHostToDevice));
  AMR_TRY(cudaMemcpy(d_bsv, base_surf_verts, sizeof(int64_t) * 2 * nbs, cudaMemcpyHostToDevice));
  AMR_TRY(cudaMemcpy(d_bcol, base_colors, sizeof(int32_t) * nbs, cudaMemcpyHostToDevice));
  k_base_keys<<<grid_for(nbs), 256>>>(d_bsv, nbs, n_base_vertices, d_key, d_sid);
  AMR_TRY(cudaGetLastError());
  AMR_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, d_key, d_key2, d_sid, d_sid2, nbs));
  AMR_TRY(cudaMalloc(&d_tmp, tmp));
  AMR_TRY(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, d_key, d_key2, d_sid, d_sid2, nbs));
  if (ns) {
    k_classify<<<grid_for(ns), 256>>>(d_fsv, ns, n_base_vertices, d_split, d_bsv, d_bcol, d_key2,
                                      d_sid2, nbs, d_org, d_bs, d_half, d_col, d_err);
    AMR_TRY(cudaGetLastError());
  }
  AMR_TRY(cudaMemcpy(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (herr) {
    rc = mc_fail(MC_EINTERNAL, herr == 2 ? "interior edge spans two parents"
                                         : "fine edge without a base counterpart");
    goto done;
  }
  if (ns) {
    AMR_TRY(cudaMemcpy(surf_origin, d_org, ns, cudaMemcpyDeviceToHost));
    AMR_TRY(cudaMemcpy(half_index, d_half, ns, cudaMemcpyDeviceToHost));
    AMR_TRY(cudaMemcpy(base_surface, d_bs, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost));
    AMR_TRY(cudaMemcpy(colors, d_col, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost));
  }
done:
  cudaFree(d_fsv);
  cudaFree(d_split);
  cudaFree(d_bsv);
  cudaFree(d_sid);
  cudaFree(d_sid2);
  cudaFree(d_key);
  cudaFree(d_key2);
  cudaFree(d_bcol);
  cudaFree(d_bs);
  cudaFree(d_col);
  cudaFree(d_org);
  cudaFree(d_half);
  cudaFree(d_err);
  cudaFree(d_tmp);
  return rc;
}

}  // extern "C"
