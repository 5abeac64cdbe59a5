// Integer Algorithm 1 on sm_100a: the colored sweep, the buffer-and-reduce
// sweep, the atomic sweep and the race certificate, behind the C ABI.
//
// Reference semantics (/root/reference/pkg/src/meshchroma/sweeps.py):
//   sweep_colored  :114-152  tot[L] += f, tot[R] -= f (R >= 0), one color at
//                            a time with a barrier between colors
//   surface_buffer :155-176  buf[2s] = f, buf[2s+1] = -f (interior) or 0
//   sweep_buffered :179-204  per element, sum its slots in local side order
//   assert_race_free :89-105 first color with a doubly written element
// Integer addition is exact and associative, so every strategy must agree
// bit for bit with sweep_sequential (sweeps.py:74-86).
//
// Device layout (one per (mesh, coloring)): surfaces grouped by color in
// ascending id order inside each color (sweeps.py:145), stored as int2
// {left, right} in that color-major order plus the original surface id.
// When the color-major order is the identity (a mesh already renumbered by
// reorder.apply_plan) the id indirection is dropped and every access of the
// color-1 block is perfectly coalesced.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "mc_internal.h"

#define MC_CUDA_TRY(expr)                                                   \
  do {                                                                      \
    cudaError_t err__ = (expr);                                             \
    if (err__ != cudaSuccess)                                               \
      return mc_fail(MC_ECUDA, std::string(#expr) + ": " +                  \
                                   cudaGetErrorString(err__));              \
  } while (0)

struct mc_layout {
  int64_t ns = 0, ne = 0;
  int n_colors = 0;
  std::vector<int64_t> bounds;   // n_colors + 1 prefix sums (host)
  bool identity = false;         // color-major order == surface-id order
  int2* d_lr = nullptr;          // color-major {left, right}
  int32_t* d_sid = nullptr;      // color-major -> original surface id
  int2* d_lr_by_id = nullptr;    // surface-id order {left, right}
  int32_t* d_elem_surfs = nullptr;  // ne x 4 (-1 padded)
  int32_t* d_counts = nullptr;   // ne scratch for the race check
  int64_t* d_race = nullptr;     // 3 x int64 scratch for the race check
  // host-path scratch
  int64_t* d_payload = nullptr;
  int64_t* d_totals = nullptr;
  int64_t* d_buffer = nullptr;
  cudaStream_t stream = nullptr;
};

namespace {

constexpr int kThreads = 256;
constexpr int kU = 4;   // surfaces per thread per iteration in k_sweep_color

inline int grid_for(int64_t n, int threads = kThreads) {
  int64_t g = (n + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(1) << 30)));
}

// ------------------------------------------------------------- kernels
template <bool kIdentity>
__global__ void __launch_bounds__(kThreads)
k_sweep_color(const int2* __restrict__ lr, const int32_t* __restrict__ sid,
              const int64_t* __restrict__ payload, int64_t* totals,
              int64_t begin, int64_t end) {
  // one color: no two surfaces share an element, so plain read-modify-write
  // is race free; that is the whole point of the coloring.  kU surfaces per
  // thread (stride = grid) with every load issued before the first store, so
  // the read-modify-write latency is paid once per kU surfaces.
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k0 = begin + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k0 < end;
       k0 += kU * stride) {
    int2 e[kU];
    int64_t v[kU], tl[kU], tr[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = k0 + u * stride;
      e[u] = k < end ? __ldg(&lr[k]) : make_int2(-1, -1);
      v[u] = k < end ? __ldg(&payload[kIdentity ? k : __ldg(&sid[k])]) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      tl[u] = e[u].x >= 0 ? totals[e[u].x] : 0;
      tr[u] = e[u].y >= 0 ? totals[e[u].y] : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (e[u].x >= 0) totals[e[u].x] = tl[u] + v[u];
      if (e[u].y >= 0) totals[e[u].y] = tr[u] - v[u];
    }
  }
}

__global__ void __launch_bounds__(kThreads)
k_sweep_atomic(const int2* __restrict__ lr, const int64_t* __restrict__ payload,
               int64_t* totals, int64_t n) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int2 e = __ldg(&lr[s]);
    const int64_t v = __ldg(&payload[s]);
    atomicAdd(reinterpret_cast<unsigned long long*>(&totals[e.x]),
              static_cast<unsigned long long>(v));
    if (e.y >= 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&totals[e.y]),
                static_cast<unsigned long long>(-v));
  }
}

__global__ void __launch_bounds__(kThreads)
k_fill_buffer(const int2* __restrict__ lr, const int64_t* __restrict__ payload,
              longlong2* buffer, int64_t n) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = __ldg(&payload[s]);
    const int2 e = __ldg(&lr[s]);
    buffer[s] = make_longlong2(v, e.y >= 0 ? -v : 0);
  }
}

__global__ void __launch_bounds__(kThreads)
k_gather_buffer(const int4* __restrict__ elem_surfs, const int2* __restrict__ lr,
                const int64_t* __restrict__ buffer, int64_t* totals, int64_t ne) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < ne;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int4 sl = __ldg(&elem_surfs[e]);
    const int ss[4] = {sl.x, sl.y, sl.z, sl.w};
    int64_t acc = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int s = ss[j];
      if (s < 0) break;  // local side order, stop at the first pad (sweeps.py:192-195)
      const int left = __ldg(&lr[s]).x;
      acc += __ldg(&buffer[2 * int64_t(s) + (left == e ? 0 : 1)]);
    }
    totals[e] = acc;
  }
}

__global__ void __launch_bounds__(kThreads)
k_race_count(const int2* __restrict__ lr, int32_t* counts, int64_t begin,
             int64_t end) {
  for (int64_t k = begin + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
       k < end; k += int64_t(gridDim.x) * blockDim.x) {
    const int2 e = __ldg(&lr[k]);
    atomicAdd(&counts[e.x], 1);
    if (e.y >= 0) atomicAdd(&counts[e.y], 1);
  }
}

__global__ void __launch_bounds__(kThreads)
k_race_first(const int32_t* __restrict__ counts, int64_t ne,
             unsigned long long* first, const int64_t* race) {
  if (race[2] != 0) return;  // an earlier color already failed
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < ne;
       e += int64_t(gridDim.x) * blockDim.x)
    if (counts[e] > 1) atomicMin(first, static_cast<unsigned long long>(e));
}

__global__ void k_race_fetch(const int32_t* __restrict__ counts,
                             int64_t* race, int color) {
  // race[0] = smallest doubly written element (or ~0), race[1] = its count,
  // race[2] = first offending color (0 = none)
  const unsigned long long first = static_cast<unsigned long long>(race[0]);
  if (race[2] == 0 && first != ~0ull) {
    race[1] = counts[first];
    race[2] = color;
  } else if (race[2] == 0) {
    race[0] = -1;
  }
}

__global__ void k_default_payload(int64_t n, uint64_t seed_term, int64_t* out) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x) {
    uint64_t z = uint64_t(k + 1) * 0x9E3779B97F4A7C15ull + seed_term;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    out[k] = int64_t(z >> 44) - (int64_t(1) << 19);
  }
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int check_launch() {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return mc_fail(MC_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(err));
  return MC_OK;
}

template <class T>
int dev_alloc(T** p, int64_t count) {
  if (count <= 0) count = 1;
  cudaError_t err = cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * size_t(count));
  if (err != cudaSuccess)
    return mc_fail(MC_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(err));
  return MC_OK;
}

int ensure_host_scratch(mc_layout* L) {
  int rc;
  if (!L->d_payload && (rc = dev_alloc(&L->d_payload, L->ns))) return rc;
  if (!L->d_totals && (rc = dev_alloc(&L->d_totals, L->ne))) return rc;
  if (!L->stream) MC_CUDA_TRY(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking));
  return MC_OK;
}

}  // namespace

extern "C" {

MC_API int mc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

MC_API int mc_layout_create(int64_t n_surfaces, int64_t n_elements,
                            const int64_t* surf_elems, const int64_t* elem_surfs,
                            const int32_t* colors, int n_colors, mc_layout** out) {
  if (!out) return mc_fail(MC_EINVAL, "null output handle");
  *out = nullptr;
  if (n_surfaces < 0 || n_elements <= 0 || n_colors < 0)
    return mc_fail(MC_EINVAL, "bad mesh sizes");
  if (n_surfaces >= (int64_t(1) << 31) || n_elements >= (int64_t(1) << 31))
    return mc_fail(MC_EINVAL, "mesh too large for 32-bit element ids");
  for (int64_t k = 0; k < n_surfaces; ++k)
    if (colors[k] < 1) return mc_fail(MC_EINVAL, "colored sweep needs a complete coloring");
  auto L = new mc_layout();
  L->ns = n_surfaces;
  L->ne = n_elements;
  L->n_colors = n_colors;
  // stable counting sort by color: ascending surface id inside each color
  std::vector<int64_t> count(n_colors + 2, 0);
  for (int64_t k = 0; k < n_surfaces; ++k)
    if (colors[k] <= n_colors) ++count[colors[k]];
  L->bounds.assign(n_colors + 1, 0);
  for (int c = 1; c <= n_colors; ++c) L->bounds[c] = L->bounds[c - 1] + count[c];
  const int64_t n_swept = L->bounds[n_colors];
  std::vector<int64_t> fill(L->bounds.begin(), L->bounds.end());
  std::vector<int32_t> sid(std::max<int64_t>(n_swept, 1));
  std::vector<int2> lr(std::max<int64_t>(n_swept, 1)), lr_id(std::max<int64_t>(n_surfaces, 1));
  bool identity = n_swept == n_surfaces;
  for (int64_t k = 0; k < n_surfaces; ++k) {
    const int64_t l = surf_elems[2 * k], r = surf_elems[2 * k + 1];
    if (l < 0 || l >= n_elements || r >= n_elements) {
      delete L;
      return mc_fail(MC_EINVAL, "surface " + std::to_string(k) + " references a bad element");
    }
    lr_id[k] = make_int2(int(l), r >= 0 ? int(r) : -1);
    const int c = colors[k];
    if (c > n_colors) continue;
    const int64_t slot = fill[c - 1]++;
    sid[slot] = int32_t(k);
    lr[slot] = lr_id[k];
    if (slot != k) identity = false;
  }
  L->identity = identity;
  std::vector<int32_t> es(size_t(n_elements) * 4, -1);
  if (elem_surfs)
    for (int64_t i = 0; i < n_elements * 4; ++i) es[i] = int32_t(elem_surfs[i]);
  int rc;
  if ((rc = dev_alloc(&L->d_lr, n_swept)) || (rc = dev_alloc(&L->d_sid, n_swept)) ||
      (rc = dev_alloc(&L->d_lr_by_id, n_surfaces)) ||
      (rc = dev_alloc(&L->d_elem_surfs, n_elements * 4)) ||
      (rc = dev_alloc(&L->d_counts, n_elements)) || (rc = dev_alloc(&L->d_race, 3))) {
    mc_layout_destroy(L);
    return rc;
  }
  cudaError_t err = cudaSuccess;
  if (n_swept) {
    err = cudaMemcpy(L->d_lr, lr.data(), sizeof(int2) * n_swept, cudaMemcpyHostToDevice);
    if (err == cudaSuccess)
      err = cudaMemcpy(L->d_sid, sid.data(), sizeof(int32_t) * n_swept, cudaMemcpyHostToDevice);
  }
  if (err == cudaSuccess && n_surfaces)
    err = cudaMemcpy(L->d_lr_by_id, lr_id.data(), sizeof(int2) * n_surfaces, cudaMemcpyHostToDevice);
  if (err == cudaSuccess)
    err = cudaMemcpy(L->d_elem_surfs, es.data(), sizeof(int32_t) * es.size(), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    mc_layout_destroy(L);
    return mc_fail(MC_ECUDA, std::string("layout upload: ") + cudaGetErrorString(err));
  }
  *out = L;
  return MC_OK;
}

MC_API int mc_layout_destroy(mc_layout* L) {
  if (!L) return MC_OK;
  cudaFree(L->d_lr);
  cudaFree(L->d_sid);
  cudaFree(L->d_lr_by_id);
  cudaFree(L->d_elem_surfs);
  cudaFree(L->d_counts);
  cudaFree(L->d_race);
  cudaFree(L->d_payload);
  cudaFree(L->d_totals);
  cudaFree(L->d_buffer);
  if (L->stream) cudaStreamDestroy(L->stream);
  delete L;
  return MC_OK;
}

MC_API int64_t mc_layout_color_size(const mc_layout* L, int color) {
  if (!L || color < 1 || color > L->n_colors) return -1;
  return L->bounds[color] - L->bounds[color - 1];
}

MC_API int mc_layout_race_check(mc_layout* L, void* stream) {
  if (!L) return mc_fail(MC_EINVAL, "null layout");
  cudaStream_t s = as_stream(stream);
  const int64_t init[3] = {-1, 0, 0};
  MC_CUDA_TRY(cudaMemcpyAsync(L->d_race, init, sizeof(init), cudaMemcpyHostToDevice, s));
  for (int c = 1; c <= L->n_colors; ++c) {
    const int64_t b = L->bounds[c - 1], e = L->bounds[c];
    if (e == b) continue;
    MC_CUDA_TRY(cudaMemsetAsync(L->d_counts, 0, sizeof(int32_t) * L->ne, s));
    k_race_count<<<grid_for(e - b), kThreads, 0, s>>>(L->d_lr, L->d_counts, b, e);
    k_race_first<<<grid_for(L->ne), kThreads, 0, s>>>(
        L->d_counts, L->ne, reinterpret_cast<unsigned long long*>(L->d_race), L->d_race);
    k_race_fetch<<<1, 1, 0, s>>>(L->d_counts, L->d_race, c);
    if (int rc = check_launch()) return rc;
  }
  int64_t res[3];
  MC_CUDA_TRY(cudaMemcpyAsync(res, L->d_race, sizeof(res), cudaMemcpyDeviceToHost, s));
  MC_CUDA_TRY(cudaStreamSynchronize(s));
  if (res[2] != 0)
    return mc_fail(MC_ECONFLICT, "color " + std::to_string(res[2]) + " writes element " +
                                     std::to_string(res[0]) + " " + std::to_string(res[1]) +
                                     " times");
  return MC_OK;
}

MC_API int mc_sweep_colored_i64(mc_layout* L, const int64_t* payload, int64_t* totals,
                                void* stream) {
  if (!L || !payload || !totals) return mc_fail(MC_EINVAL, "null argument");
  cudaStream_t s = as_stream(stream);
  MC_CUDA_TRY(cudaMemsetAsync(totals, 0, sizeof(int64_t) * L->ne, s));
  for (int c = 1; c <= L->n_colors; ++c) {
    const int64_t b = L->bounds[c - 1], e = L->bounds[c];
    if (e == b) continue;
    if (L->identity)
      k_sweep_color<true><<<grid_for((e - b + kU - 1) / kU), kThreads, 0, s>>>(L->d_lr, L->d_sid, payload, totals, b, e);
    else
      k_sweep_color<false><<<grid_for((e - b + kU - 1) / kU), kThreads, 0, s>>>(L->d_lr, L->d_sid, payload, totals, b, e);
  }
  return check_launch();
}

MC_API int mc_surface_buffer_i64(mc_layout* L, const int64_t* payload, int64_t* buffer,
                                 void* stream) {
  if (!L || !payload || !buffer) return mc_fail(MC_EINVAL, "null argument");
  if (L->ns == 0) return MC_OK;
  k_fill_buffer<<<grid_for(L->ns), kThreads, 0, as_stream(stream)>>>(
      L->d_lr_by_id, payload, reinterpret_cast<longlong2*>(buffer), L->ns);
  return check_launch();
}

MC_API int mc_sweep_buffered_i64(mc_layout* L, const int64_t* payload, int64_t* buffer,
                                 int64_t* totals, void* stream) {
  if (int rc = mc_surface_buffer_i64(L, payload, buffer, stream)) return rc;
  // stream order is the barrier between the fill and the gather
  k_gather_buffer<<<grid_for(L->ne), kThreads, 0, as_stream(stream)>>>(
      reinterpret_cast<const int4*>(L->d_elem_surfs), L->d_lr_by_id, buffer, totals, L->ne);
  return check_launch();
}

MC_API int mc_sweep_atomic_i64(mc_layout* L, const int64_t* payload, int64_t* totals,
                               void* stream) {
  if (!L || !payload || !totals) return mc_fail(MC_EINVAL, "null argument");
  cudaStream_t s = as_stream(stream);
  MC_CUDA_TRY(cudaMemsetAsync(totals, 0, sizeof(int64_t) * L->ne, s));
  if (L->ns)
    k_sweep_atomic<<<grid_for(L->ns), kThreads, 0, s>>>(L->d_lr_by_id, payload, totals, L->ns);
  return check_launch();
}

MC_API int mc_sweep_i64_host(mc_layout* L, int strategy, const int64_t* payload_host,
                             int64_t* totals_host) {
  if (!L || !payload_host || !totals_host) return mc_fail(MC_EINVAL, "null argument");
  if (int rc = ensure_host_scratch(L)) return rc;
  cudaStream_t s = L->stream;
  MC_CUDA_TRY(cudaMemcpyAsync(L->d_payload, payload_host, sizeof(int64_t) * L->ns,
                              cudaMemcpyHostToDevice, s));
  int rc;
  if (strategy == 0) {
    rc = mc_sweep_colored_i64(L, L->d_payload, L->d_totals, s);
  } else if (strategy == 1) {
    if (!L->d_buffer && (rc = dev_alloc(&L->d_buffer, 2 * L->ns))) return rc;
    rc = mc_sweep_buffered_i64(L, L->d_payload, L->d_buffer, L->d_totals, s);
  } else if (strategy == 2) {
    rc = mc_sweep_atomic_i64(L, L->d_payload, L->d_totals, s);
  } else {
    return mc_fail(MC_EINVAL, "unknown sweep strategy");
  }
  if (rc) return rc;
  MC_CUDA_TRY(cudaMemcpyAsync(totals_host, L->d_totals, sizeof(int64_t) * L->ne,
                              cudaMemcpyDeviceToHost, s));
  MC_CUDA_TRY(cudaStreamSynchronize(s));
  return MC_OK;
}

MC_API int mc_default_payload_dev(int64_t n, int64_t seed, int64_t* out, void* stream) {
  if (n < 0 || (n && !out)) return mc_fail(MC_EINVAL, "bad payload arguments");
  if (n == 0) return MC_OK;
  const uint64_t seed_term = uint64_t(seed) * 0x94D049BB133111EBull;  // (seed*MIX2) mod 2^64
  k_default_payload<<<grid_for(n), kThreads, 0, as_stream(stream)>>>(n, seed_term, out);
  return check_launch();
}

}  // extern "C"
