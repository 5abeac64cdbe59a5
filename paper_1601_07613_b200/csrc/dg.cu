// C ABI of the DG operator: handle creation (upload of the color-major
// surface list, element geometry and reference tables), the colored /
// buffered / atomic RHS strategies and the fused SSP-RK3 stepper.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "dg_ops.h"
#include "mc_internal.h"

using mcdg::Ops;

struct mc_dg {
  Ops* ops = nullptr;
  mcdg::View view{};
  int n_colors = 0;
  std::vector<int64_t> bounds;
  std::vector<char> has_first, has_last;   // per color: any first / last touch
  int64_t ne = 0, ng = 0, ns = 0, stride = 0;
  // device allocations
  int32_t *d_left = nullptr, *d_right = nullptr, *d_slots = nullptr;
  uint32_t* d_code = nullptr;
  uint8_t* d_ekind = nullptr;      // MC_KIND_HYBRID: element kinds (0 tri, 1 quad)
  double *d_geom = nullptr, *d_jinv = nullptr, *d_tables = nullptr, *d_ptables = nullptr;
  int64_t* d_slot_ptr = nullptr;
  double* d_buffer = nullptr;      // 2*ns blocks (buffered strategy)
  char* d_host_U = nullptr;        // host path scratch: U, U0, R (state type)
  int f32 = 0;                     // fp32 state storage (element blocks of floats)
  int64_t esize = 8;               // bytes per state value
  cudaStream_t stream = nullptr;
  // one SSP-RK3 step captured as a CUDA graph (9-12 launches replayed with
  // one cudaGraphLaunch), keyed by the arguments baked into it
  cudaGraphExec_t step_exec = nullptr;
  double *g_U = nullptr, *g_work = nullptr;
  double g_dt = 0.0;
  cudaStream_t g_stream = nullptr;
  // upper bound on the blocks of every persistent-grid launch (0 = none):
  // lets tests make each warp loop over many tiles on a small mesh
  int grid_cap = 0;
  // caller (user) element order: internal owned row r <- user row src[r]
  int64_t* d_user_src = nullptr;
  int64_t n_user_rows = 0;
  double* d_user = nullptr;        // user-layout staging (n_user_rows x W)
  double* d_user_R = nullptr;      // user-layout residual staging
  int32_t* d_send_slot = nullptr;  // per owned element: ghost send-buffer slot or -1
  int64_t* d_push_ptr = nullptr;   // peer push: CSR of destinations per owned element
  unsigned long long* d_push_dst = nullptr;
};

namespace {

#define DG_TRY(expr)                                                                    \
  do {                                                                                  \
    cudaError_t e__ = (expr);                                                           \
    if (e__ != cudaSuccess)                                                             \
      return mc_fail(MC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));    \
  } while (0)

template <class T>
cudaError_t upload(T** dst, const T* src, int64_t count) {
  if (count <= 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), sizeof(T) * size_t(count));
  if (e != cudaSuccess) return e;
  if (src) return cudaMemcpy(*dst, src, sizeof(T) * size_t(count), cudaMemcpyHostToDevice);
  return cudaSuccess;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// `blocks` element blocks past `base` in the operator's state type
template <class P>
P* at_blocks(P* base, const mc_dg* h, int64_t blocks) {
  using B = typename std::conditional<std::is_const<P>::value, const char, char>::type;
  return reinterpret_cast<P*>(reinterpret_cast<B*>(base) + blocks * h->stride * h->esize);
}

int colored_grid(const mc_dg* h, int64_t n, int variant) {
  // never launch more warps than surface tiles of the color
  const int64_t tiles = (n + h->ops->spw - 1) / h->ops->spw;
  const int64_t wpb = h->ops->threads / 32;
  const int64_t max_blocks = (tiles + wpb - 1) / wpb;
  // MC_MIN_GRID=1: every variant at the smallest resident grid (round 1)
  static const bool min_grid = std::getenv("MC_MIN_GRID") != nullptr;
  int grid = min_grid ? h->ops->grid_colored : h->ops->grid_var[variant & 3];
  static const bool full = std::getenv("MC_FULL_GRID") != nullptr;   // A/B knob
  if (full || grid > max_blocks) grid = int(std::min<int64_t>(max_blocks, 1 << 30));
  if (h->grid_cap > 0 && grid > h->grid_cap) grid = h->grid_cap;
  return grid < 1 ? 1 : grid;
}

int capped(const mc_dg* h, int grid) {
  return (h->grid_cap > 0 && grid > h->grid_cap) ? h->grid_cap : grid;
}

// user layout (n_user_rows x W, W = N_eq*N_p doubles per element, caller
// order) <-> internal layout (renumbered rows, `stride`-padded blocks); one
// thread per internal double, coalesced on the internal side, W contiguous
// doubles per row on the user side
template <class S>
__global__ void k_user_to_internal(const double* __restrict__ user, const int64_t* __restrict__ src,
                                   S* __restrict__ U, int64_t rows, int W, int stride) {
  const int64_t total = rows * stride;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / stride;
    const int j = int(i - r * stride);
    U[i] = S(j < W ? __ldg(user + __ldg(src + r) * W + j) : 0.0);
  }
}

template <class S>
__global__ void k_internal_to_user(const S* __restrict__ U, const int64_t* __restrict__ src,
                                   double* __restrict__ user, int64_t rows, int W, int stride) {
  const int64_t total = rows * W;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / W;
    const int j = int(i - r * W);
    user[__ldg(src + r) * W + j] = double(U[r * stride + j]);
  }
}

int copy_grid(int64_t total) {
  const int64_t g = (total + 255) / 256;
  return int(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16)));
}

// Tables of the projection through P_{p-1} (dg_kernels.cuh Cfg::NPL):
// WPSI[q][m] = w_q phi_m(q) and D_r[j][m] with dphi_r[q][j] =
// sum_m D_r[j][m] phi_m(q), fitted by least squares on the volume points
// (the representation is exact: the fit residual is rounding).  Also checks
// the hierarchical mode order the kernels' sparsity relies on.
int p1_tables(const Ops* ops, const mc_dg_desc* d, double* out) {
  const int M = ops->npl, nq = ops->nqv, np = ops->np, dim = ops->dim;
  double* wpsi = out;
  double* dmat = out + nq * M;
  for (int q = 0; q < nq; ++q)
    for (int m = 0; m < M; ++m) wpsi[q * M + m] = d->vol_w[q] * d->vol_phi[q * np + m];
  // normal equations A^T A x = A^T b, A = phi[:, :M] (long double Gauss-Jordan)
  std::vector<long double> ata(M * M, 0.0L), inv(M * M, 0.0L);
  for (int a = 0; a < M; ++a)
    for (int b = 0; b < M; ++b)
      for (int q = 0; q < nq; ++q)
        ata[a * M + b] += (long double)d->vol_phi[q * np + a] * d->vol_phi[q * np + b];
  for (int a = 0; a < M; ++a) inv[a * M + a] = 1.0L;
  for (int c = 0; c < M; ++c) {
    int piv = c;
    for (int r = c + 1; r < M; ++r)
      if (std::fabs((double)ata[r * M + c]) > std::fabs((double)ata[piv * M + c])) piv = r;
    if (std::fabs((double)ata[piv * M + c]) < 1e-12)
      return mc_fail(MC_EINVAL, "volume points do not determine the P_{p-1} modes");
    for (int k = 0; k < M; ++k) {
      std::swap(ata[c * M + k], ata[piv * M + k]);
      std::swap(inv[c * M + k], inv[piv * M + k]);
    }
    const long double f = 1.0L / ata[c * M + c];
    for (int k = 0; k < M; ++k) {
      ata[c * M + k] *= f;
      inv[c * M + k] *= f;
    }
    for (int r = 0; r < M; ++r)
      if (r != c) {
        const long double g = ata[r * M + c];
        for (int k = 0; k < M; ++k) {
          ata[r * M + k] -= g * ata[c * M + k];
          inv[r * M + k] -= g * inv[c * M + k];
        }
      }
  }
  // shell of mode j: number of P_{deg(j)-1} modes (0 for the constant)
  auto nsimp = [&](int deg) {
    if (deg < 0) return 0;
    return dim == 2 ? (deg + 1) * (deg + 2) / 2 : (deg + 1) * (deg + 2) * (deg + 3) / 6;
  };
  for (int r = 0; r < dim; ++r)
    for (int j = 0; j < np; ++j) {
      std::vector<long double> atb(M, 0.0L);
      for (int m = 0; m < M; ++m)
        for (int q = 0; q < nq; ++q)
          atb[m] += (long double)d->vol_phi[q * np + m] * d->vol_dphi[(r * nq + q) * np + j];
      int deg = 0;
      while (j >= nsimp(deg)) ++deg;
      const int shell = nsimp(deg - 1);
      double resid = 0.0;
      for (int m = 0; m < M; ++m) {
        long double x = 0.0L;
        for (int k = 0; k < M; ++k) x += inv[m * M + k] * atb[k];
        dmat[(r * np + j) * M + m] = double(x);
        if (m >= shell) resid = std::max(resid, std::fabs(double(x)));
      }
      if (ops->p1proj && resid > 1e-9)
        return mc_fail(MC_EINVAL, "basis modes are not ordered by total degree");
    }
  return MC_OK;
}

int colored_pass(mc_dg* h, void* U, void* R, const mcdg::RK* rk, cudaStream_t s) {
  for (int c = 1; c <= h->n_colors; ++c) {
    const int64_t b = h->bounds[c - 1], e = h->bounds[c];
    if (e == b) continue;
    const int variant = ((rk && h->has_last[c]) ? 2 : 0) | (h->has_first[c] ? 1 : 0);
    DG_TRY(h->ops->colored(h->view, U, R, rk, b, e, colored_grid(h, e - b, variant), s,
                           h->has_first[c], h->has_last[c], h->f32));
  }
  return MC_OK;
}

}  // namespace

extern "C" {

MC_API int mc_dg_create(const mc_dg_desc* d, mc_dg** out) {
  if (!d || !out) return mc_fail(MC_EINVAL, "null argument");
  *out = nullptr;
  Ops* ops = nullptr;
  if (d->kind == MC_KIND_TRI) ops = mcdg::ops_tri(d->physics, d->degree);
  else if (d->kind == MC_KIND_QUAD) ops = mcdg::ops_quad(d->physics, d->degree);
  else if (d->kind == MC_KIND_TET) ops = mcdg::ops_tet(d->physics, d->degree);
  else if (d->kind == MC_KIND_HYBRID) ops = mcdg::ops_hyb(d->physics, d->degree);
  if (!ops)
    return mc_fail(MC_EUNSUPPORTED, "no sm_100a kernel compiled for kind " +
                                        std::to_string(d->kind) + " physics " +
                                        std::to_string(d->physics) + " degree " +
                                        std::to_string(d->degree));
  if (d->n_face_codes != ops->ncodes || d->n_face_q != ops->nqf || d->n_vol_q != ops->nqv ||
      d->n_basis != ops->np)
    return mc_fail(MC_EINVAL, "reference tables do not match the compiled kernel");
  if (d->state_f32 && !ops->tpe)
    return mc_fail(MC_EUNSUPPORTED, "fp32 state needs the register kernels (N_eq * N_p <= 64)");
  if (d->n_elements <= 0 || d->n_surfaces < 0 || d->n_colors < 1 || d->n_ghosts < 0)
    return mc_fail(MC_EINVAL, "bad DG sizes");
  if (d->kind == MC_KIND_HYBRID) {
    if (!d->elem_kind) return mc_fail(MC_EINVAL, "hybrid mesh without element kinds");
    for (int64_t i = 0; i < d->n_elements + d->n_ghosts; ++i)
      if (d->elem_kind[i] > 1)
        return mc_fail(MC_EINVAL, "element " + std::to_string(i) + " kind must be 0 or 1");
  }
  if (d->n_elements + d->n_ghosts >= (int64_t(1) << 31) || d->n_surfaces >= (int64_t(1) << 31))
    return mc_fail(MC_EINVAL, "mesh too large for 32-bit ids");
  if (d->group_bounds[0] != 0 || d->group_bounds[d->n_colors] != d->n_surfaces)
    return mc_fail(MC_EINVAL, "group bounds do not cover the surface list");
  for (int c = 1; c <= d->n_colors; ++c)
    if (d->group_bounds[c] < d->group_bounds[c - 1])
      return mc_fail(MC_EINVAL, "group bounds must be non-decreasing");
  const int64_t nall = d->n_elements + d->n_ghosts;
  for (int64_t s = 0; s < d->n_surfaces; ++s) {
    const int32_t l = d->surf_left[s], r = d->surf_right[s];
    if (l < 0 || l >= d->n_elements || r >= nall)
      return mc_fail(MC_EINVAL, "surface " + std::to_string(s) + " has a bad element id");
  }
  if (ops->init) {
    cudaError_t e = ops->init(ops);
    ops->init = nullptr;  // once per process
    if (e != cudaSuccess)
      return mc_fail(MC_ECUDA, std::string("kernel setup: ") + cudaGetErrorString(e));
  }
  if (const char* g = std::getenv("MC_L2_FETCH")) {  // experiment knob (bytes)
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(std::atoi(g)));
  }
  auto h = new mc_dg();
  h->ops = ops;
  h->n_colors = d->n_colors;
  h->bounds.assign(d->group_bounds, d->group_bounds + d->n_colors + 1);
  h->has_first.assign(d->n_colors + 1, 0);
  h->has_last.assign(d->n_colors + 1, 0);
  for (int c = 1; c <= d->n_colors; ++c)
    for (int64_t s = h->bounds[c - 1]; s < h->bounds[c]; ++s) {
      const uint32_t code = d->surf_code[s];
      if (code & (MC_FLAG_L_FIRST | MC_FLAG_R_FIRST)) h->has_first[c] = 1;
      if (code & (MC_FLAG_L_LAST | MC_FLAG_R_LAST)) h->has_last[c] = 1;
    }
  h->ne = d->n_elements;
  h->ng = d->n_ghosts;
  h->ns = d->n_surfaces;
  const int64_t w = int64_t(ops->neq) * ops->np;
  // 32-byte aligned element blocks; MC_BLOCK_ALIGN=<doubles> (a multiple of
  // 4) pads further, for DRAM-atom experiments (c4: 52 -> 56 doubles)
  int64_t align = 4;
  if (const char* a = std::getenv("MC_BLOCK_ALIGN")) align = std::max<int64_t>(4, std::atoi(a) / 4 * 4);
  h->stride = (w + align - 1) / align * align;   // fp32 state: 4 floats = 16-byte aligned
  h->f32 = d->state_f32 ? 1 : 0;
  h->esize = h->f32 ? 4 : 8;
  const int dim = ops->dim;
  std::vector<double> tables(ops->table_size);
  {
    double* t = tables.data();
    const int64_t nf = int64_t(ops->ncodes) * ops->nqf * ops->np;
    std::memcpy(t, d->face_phi, sizeof(double) * nf);
    t += nf;
    std::memcpy(t, d->face_w, sizeof(double) * ops->nqf);
    t += ops->nqf;
    std::memcpy(t, d->vol_phi, sizeof(double) * ops->nqv * ops->np);
    t += ops->nqv * ops->np;
    std::memcpy(t, d->vol_dphi, sizeof(double) * dim * ops->nqv * ops->np);
    t += dim * ops->nqv * ops->np;
    std::memcpy(t, d->vol_w, sizeof(double) * ops->nqv);
    t += ops->nqv;
    if (int rc = p1_tables(ops, d, t)) {
      delete h;
      return rc;
    }
  }
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = upload(&h->d_left, d->surf_left, h->ns);
  if (e == cudaSuccess) e = upload(&h->d_right, d->surf_right, h->ns);
  if (e == cudaSuccess) e = upload(&h->d_code, d->surf_code, h->ns);
  if (e == cudaSuccess) e = upload(&h->d_geom, d->surf_geom, h->ns * (dim + 2));
  if (e == cudaSuccess) e = upload(&h->d_jinv, d->elem_jinv, nall * dim * dim);
  if (e == cudaSuccess && d->kind == MC_KIND_HYBRID) e = upload(&h->d_ekind, d->elem_kind, nall);
  if (e == cudaSuccess) e = upload(&h->d_tables, tables.data(), int64_t(tables.size()));
  if (e == cudaSuccess && d->elem_slot_ptr) e = upload(&h->d_slot_ptr, d->elem_slot_ptr, h->ne + 1);
  if (e == cudaSuccess && d->elem_slots)
    e = upload(&h->d_slots, d->elem_slots, d->elem_slot_ptr[h->ne]);
  if (e != cudaSuccess) {
    mc_dg_destroy(h);
    return mc_fail(MC_ENOMEM, std::string("DG upload: ") + cudaGetErrorString(e));
  }
  if (e == cudaSuccess) e = cudaMalloc(&h->d_ptables, sizeof(double) * size_t(ops->stable_size));
  if (e == cudaSuccess) e = ops->stage_global(h->d_tables, h->d_ptables, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = ops->upload_const(h->d_ptables);
  if (e != cudaSuccess) {
    mc_dg_destroy(h);
    return mc_fail(MC_ECUDA, std::string("DG table staging: ") + cudaGetErrorString(e));
  }
  mcdg::View& v = h->view;
  v.ptables = h->d_ptables;
  v.left = h->d_left;
  v.right = h->d_right;
  v.code = h->d_code;
  v.geom = h->d_geom;
  v.jinv = h->d_jinv;
  v.ekind = h->d_ekind;
  v.ghost_par = -1;
  v.tables = h->d_tables;
  v.slot_ptr = h->d_slot_ptr;
  v.slots = h->d_slots;
  v.n_elements = h->ne;
  v.n_surfaces = h->ns;
  v.stride = h->stride;
  v.prm.gamma = d->gamma;
  for (int k = 0; k < 3; ++k) v.prm.vel[k] = d->velocity[k];
  for (int k = 0; k < 5; ++k) v.prm.ff[k] = d->farfield[k];
  *out = h;
  return MC_OK;
}

MC_API int mc_dg_destroy(mc_dg* h) {
  if (!h) return MC_OK;
  cudaFree(h->d_left);
  cudaFree(h->d_right);
  cudaFree(h->d_code);
  cudaFree(h->d_geom);
  cudaFree(h->d_jinv);
  cudaFree(h->d_ekind);
  cudaFree(h->d_tables);
  cudaFree(h->d_ptables);
  cudaFree(h->d_slot_ptr);
  cudaFree(h->d_slots);
  cudaFree(h->d_buffer);
  cudaFree(h->d_host_U);
  cudaFree(h->d_user_src);
  cudaFree(h->d_user);
  cudaFree(h->d_user_R);
  cudaFree(h->d_send_slot);
  cudaFree(h->d_push_ptr);
  cudaFree(h->d_push_dst);
  if (h->step_exec) cudaGraphExecDestroy(h->step_exec);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return MC_OK;
}

MC_API int64_t mc_dg_block_stride(const mc_dg* h) { return h ? h->stride : -1; }

MC_API int mc_dg_set_grid_cap(mc_dg* h, int max_blocks) {
  if (!h || max_blocks < 0) return mc_fail(MC_EINVAL, "bad argument");
  h->grid_cap = max_blocks;
  if (h->step_exec) {   // the captured step baked the old grid sizes in
    cudaGraphExecDestroy(h->step_exec);
    h->step_exec = nullptr;
  }
  return MC_OK;
}

MC_API int64_t mc_dg_buffer_bytes(const mc_dg* h) {
  return h ? 2 * h->ns * h->stride * int64_t(sizeof(double)) : -1;   // fp64 buffer
}

MC_API int mc_dg_rhs(mc_dg* h, const double* U, double* R, int strategy, void* stream) {
  if (!h || !U || !R) return mc_fail(MC_EINVAL, "null argument");
  cudaStream_t s = as_stream(stream);
  double* Um = const_cast<double*>(U);  // the non-RK colored pass never writes U
  if (strategy == MC_DG_COLORED) return colored_pass(h, Um, R, nullptr, s);
  if (strategy != MC_DG_BUFFERED && strategy != MC_DG_ATOMIC)
    return mc_fail(MC_EINVAL, "unknown strategy");
  if (h->f32)
    return mc_fail(MC_EUNSUPPORTED, "the buffered / atomic strategies need fp64 state");
  const int gv = capped(h, h->ops->grid_volume), gu = capped(h, h->ops->grid_uncolored);
  DG_TRY(h->ops->volume(h->view, U, R, gv, s));
  if (strategy == MC_DG_ATOMIC) {
    if (h->ns) DG_TRY(h->ops->uncolored(h->view, U, R, true, gu, s));
    return MC_OK;
  }
  if (!h->d_slot_ptr) return mc_fail(MC_EINVAL, "buffered strategy needs the element slot CSR");
  if (!h->d_buffer) DG_TRY(cudaMalloc(&h->d_buffer, size_t(mc_dg_buffer_bytes(h)) + 16));
  if (h->ns) DG_TRY(h->ops->uncolored(h->view, U, h->d_buffer, false, gu, s));
  DG_TRY(h->ops->gather(h->view, h->d_buffer, R, h->grid_cap, s));
  return MC_OK;
}

MC_API int mc_dg_rk_stage(mc_dg* h, double* U, const double* U0, double* R, double a, double b,
                          double dt, void* stream) {
  if (!h || !U || !R || (a != 0.0 && !U0)) return mc_fail(MC_EINVAL, "null argument");
  mcdg::RK rk{const_cast<double*>(U0), a, b, dt, 0};
  return colored_pass(h, U, R, &rk, as_stream(stream));
}

MC_API int mc_dg_color_range_pass(mc_dg* h, int color, int64_t begin, int64_t end, double* U,
                                  double* U0, double* R, int rk_mode, double a, double b,
                                  double dt, void* stream) {
  if (!h || !U || !R) return mc_fail(MC_EINVAL, "null argument");
  if (color < 1 || color > h->n_colors) return mc_fail(MC_EINVAL, "bad color");
  const int64_t c0 = h->bounds[color - 1], c1 = h->bounds[color];
  if (begin < 0 || end < begin || c0 + end > c1) return mc_fail(MC_EINVAL, "bad surface range");
  const int64_t bb = c0 + begin, e = c0 + end;
  if (e == bb) return MC_OK;
  const int grid = colored_grid(h, e - bb, (rk_mode && h->has_last[color] ? 2 : 0) |
                                               (h->has_first[color] ? 1 : 0));
  if (rk_mode == 0) {
    DG_TRY(h->ops->colored(h->view, U, R, nullptr, bb, e, grid, as_stream(stream),
                           h->has_first[color], h->has_last[color], h->f32));
  } else {
    if (!U0) return mc_fail(MC_EINVAL, "RK pass needs U0");
    mcdg::RK rk{U0, a, b, dt, rk_mode == 2 ? 1 : 0};
    DG_TRY(h->ops->colored(h->view, U, R, &rk, bb, e, grid, as_stream(stream),
                           h->has_first[color], h->has_last[color], h->f32));
  }
  return MC_OK;
}

MC_API int mc_dg_color_pass(mc_dg* h, int color, double* U, double* U0, double* R, int rk_mode,
                            double a, double b, double dt, void* stream) {
  if (!h) return mc_fail(MC_EINVAL, "null argument");
  if (color < 1 || color > h->n_colors) return mc_fail(MC_EINVAL, "bad color");
  return mc_dg_color_range_pass(h, color, 0, h->bounds[color] - h->bounds[color - 1], U, U0, R,
                                rk_mode, a, b, dt, stream);
}

MC_API int mc_dg_ssprk3(mc_dg* h, double* U, double* work, double dt, int n_steps,
                        void* stream) {
  if (!h || !U || !work || n_steps < 0) return mc_fail(MC_EINVAL, "bad argument");
  cudaStream_t s = as_stream(stream);
  double* U0 = work;
  double* R = at_blocks(work, h, h->ne + h->ng);
  auto one_step = [&]() -> int {
    // stage 1 saves U0 := U in its last-touch pass (no separate copy)
    mcdg::RK r1{U0, 0.0, 1.0, dt, 1};
    if (int rc = colored_pass(h, U, R, &r1, s)) return rc;
    mcdg::RK r2{U0, 0.75, 0.25, dt, 0};
    if (int rc = colored_pass(h, U, R, &r2, s)) return rc;
    mcdg::RK r3{U0, 1.0 / 3.0, 2.0 / 3.0, dt, 0};
    return colored_pass(h, U, R, &r3, s);
  };
  // CUDA graph of one step on a non-default stream (capture is not allowed
  // on the legacy stream); MC_NO_GRAPH=1 launches kernel by kernel
  static const bool no_graph = std::getenv("MC_NO_GRAPH") != nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const bool graphable = !no_graph && s != nullptr && n_steps > 0 &&
                         cudaStreamIsCapturing(s, &cap) == cudaSuccess &&
                         cap == cudaStreamCaptureStatusNone;
  if (!graphable) {
    for (int step = 0; step < n_steps; ++step)
      if (int rc = one_step()) return rc;
    return MC_OK;
  }
  if (!h->step_exec || h->g_U != U || h->g_work != work || h->g_dt != dt || h->g_stream != s) {
    cudaGraph_t g = nullptr;
    DG_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const int rc = one_step();
    const cudaError_t ec = cudaStreamEndCapture(s, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ec != cudaSuccess) return mc_fail(MC_ECUDA, std::string("step capture: ") + cudaGetErrorString(ec));
    if (h->step_exec) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(h->step_exec, g, &info) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphExecDestroy(h->step_exec);
        h->step_exec = nullptr;
      }
    }
    cudaError_t ei = cudaSuccess;
    if (!h->step_exec) ei = cudaGraphInstantiate(&h->step_exec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) {
      h->step_exec = nullptr;
      return mc_fail(MC_ECUDA, std::string("step graph: ") + cudaGetErrorString(ei));
    }
    h->g_U = U;
    h->g_work = work;
    h->g_dt = dt;
    h->g_stream = s;
  }
  for (int step = 0; step < n_steps; ++step) DG_TRY(cudaGraphLaunch(h->step_exec, s));
  return MC_OK;
}

MC_API int mc_dg_ssprk3_host(mc_dg* h, double* U_host, double dt, int n_steps) {
  if (!h || !U_host) return mc_fail(MC_EINVAL, "null argument");
  const int64_t nblk = h->ne + h->ng;
  const size_t sbytes = size_t(nblk * h->stride * h->esize);
  if (!h->d_host_U) DG_TRY(cudaMalloc(&h->d_host_U, 3 * sbytes));
  if (!h->stream) DG_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  DG_TRY(cudaMemcpyAsync(h->d_host_U, U_host, sbytes, cudaMemcpyHostToDevice, h->stream));
  double* Ud = reinterpret_cast<double*>(h->d_host_U);
  if (int rc = mc_dg_ssprk3(h, Ud, at_blocks(Ud, h, nblk), dt, n_steps, h->stream)) return rc;
  DG_TRY(cudaMemcpyAsync(U_host, h->d_host_U, size_t(h->ne * h->stride * h->esize),
                         cudaMemcpyDeviceToHost, h->stream));
  DG_TRY(cudaStreamSynchronize(h->stream));
  return MC_OK;
}

MC_API int mc_dg_set_user_rows(mc_dg* h, const int64_t* src, int64_t n_user_rows) {
  if (!h || !src || n_user_rows < 1) return mc_fail(MC_EINVAL, "bad argument");
  for (int64_t r = 0; r < h->ne; ++r)
    if (src[r] < 0 || src[r] >= n_user_rows)
      return mc_fail(MC_EINVAL, "user row " + std::to_string(src[r]) + " out of range");
  cudaFree(h->d_user_src);
  cudaFree(h->d_user);
  cudaFree(h->d_user_R);
  h->d_user = h->d_user_R = nullptr;
  h->d_user_src = nullptr;
  h->n_user_rows = 0;
  DG_TRY(upload(&h->d_user_src, src, h->ne));
  h->n_user_rows = n_user_rows;
  return MC_OK;
}

MC_API int mc_dg_set_send_rows(mc_dg* h, const int32_t* slot, double* send_buf_dev,
                                int64_t n_slots) {
  if (!h) return mc_fail(MC_EINVAL, "null argument");
  cudaFree(h->d_send_slot);
  h->d_send_slot = nullptr;
  h->view.send_slot = nullptr;
  h->view.send_buf = nullptr;
  if (h->step_exec) {   // the captured step baked the old view in
    cudaGraphExecDestroy(h->step_exec);
    h->step_exec = nullptr;
  }
  if (!slot) return MC_OK;
  if (!send_buf_dev) return mc_fail(MC_EINVAL, "send buffer missing");
  for (int64_t e = 0; e < h->ne; ++e)
    if (slot[e] < -1 || slot[e] >= n_slots)
      return mc_fail(MC_EINVAL, "send slot out of range");
  DG_TRY(upload(&h->d_send_slot, slot, h->ne));
  h->view.send_slot = h->d_send_slot;
  h->view.send_buf = send_buf_dev;
  return MC_OK;
}

MC_API int mc_dg_set_push_rows(mc_dg* h, const int64_t* ptr, const uint64_t* dst, int64_t nnz) {
  if (!h) return mc_fail(MC_EINVAL, "null argument");
  cudaFree(h->d_push_ptr);
  cudaFree(h->d_push_dst);
  h->d_push_ptr = nullptr;
  h->d_push_dst = nullptr;
  h->view.push_ptr = nullptr;
  h->view.push_dst = nullptr;
  if (h->step_exec) {
    cudaGraphExecDestroy(h->step_exec);
    h->step_exec = nullptr;
  }
  if (!ptr) return MC_OK;
  if (!h->ops->tpe) return mc_fail(MC_EUNSUPPORTED, "peer push needs the register kernels");
  if (ptr[0] != 0 || ptr[h->ne] != nnz || nnz < 0)
    return mc_fail(MC_EINVAL, "push CSR does not cover the destinations");
  for (int64_t e = 0; e < h->ne; ++e)
    if (ptr[e + 1] < ptr[e]) return mc_fail(MC_EINVAL, "push CSR must be non-decreasing");
  const uint64_t align = h->f32 ? 16 : 32;
  for (int64_t k = 0; k < nnz; ++k)
    if (!dst[k] || dst[k] % align)
      return mc_fail(MC_EINVAL, "push destination " + std::to_string(k) + " is null or misaligned");
  DG_TRY(upload(&h->d_push_ptr, ptr, h->ne + 1));
  DG_TRY(upload(&h->d_push_dst, reinterpret_cast<const unsigned long long*>(dst), nnz));
  h->view.push_ptr = h->d_push_ptr;
  h->view.push_dst = h->d_push_dst;
  return MC_OK;
}

MC_API int mc_dg_set_ghost_parity(mc_dg* h, int read_parity, int push_parity) {
  if (!h) return mc_fail(MC_EINVAL, "null argument");
  if (read_parity < -1 || read_parity > 1 || push_parity < 0 || push_parity > 1)
    return mc_fail(MC_EINVAL, "parities must be -1/0/1 (read) and 0/1 (push)");
  h->view.ghost_par = read_parity;
  h->view.push_shift = int64_t(push_parity) * h->stride;
  return MC_OK;
}

MC_API int mc_dg_user_to_internal(mc_dg* h, const double* user_dev, double* U_dev, void* stream) {
  if (!h || !user_dev || !U_dev) return mc_fail(MC_EINVAL, "null argument");
  if (!h->d_user_src) return mc_fail(MC_EINVAL, "user row map not set (mc_dg_set_user_rows)");
  const int W = h->ops->neq * h->ops->np;
  if (h->f32)
    k_user_to_internal<float><<<copy_grid(h->ne * h->stride), 256, 0, as_stream(stream)>>>(
        user_dev, h->d_user_src, reinterpret_cast<float*>(U_dev), h->ne, W, int(h->stride));
  else
    k_user_to_internal<double><<<copy_grid(h->ne * h->stride), 256, 0, as_stream(stream)>>>(
        user_dev, h->d_user_src, U_dev, h->ne, W, int(h->stride));
  DG_TRY(cudaGetLastError());
  return MC_OK;
}

MC_API int mc_dg_internal_to_user(mc_dg* h, const double* U_dev, double* user_dev, void* stream) {
  if (!h || !user_dev || !U_dev) return mc_fail(MC_EINVAL, "null argument");
  if (!h->d_user_src) return mc_fail(MC_EINVAL, "user row map not set (mc_dg_set_user_rows)");
  const int W = h->ops->neq * h->ops->np;
  if (h->f32)
    k_internal_to_user<float><<<copy_grid(h->ne * W), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const float*>(U_dev), h->d_user_src, user_dev, h->ne, W, int(h->stride));
  else
    k_internal_to_user<double><<<copy_grid(h->ne * W), 256, 0, as_stream(stream)>>>(
        U_dev, h->d_user_src, user_dev, h->ne, W, int(h->stride));
  DG_TRY(cudaGetLastError());
  return MC_OK;
}

namespace {
int user_staging(mc_dg* h, bool residual) {
  if (!h->d_user_src) return mc_fail(MC_EINVAL, "user row map not set (mc_dg_set_user_rows)");
  const size_t sbytes = size_t((h->ne + h->ng) * h->stride * h->esize);
  const size_t ubytes = sizeof(double) * size_t(h->n_user_rows) * h->ops->neq * h->ops->np;
  if (!h->d_host_U) DG_TRY(cudaMalloc(&h->d_host_U, 3 * sbytes));
  if (!h->d_user) DG_TRY(cudaMalloc(&h->d_user, ubytes));
  if (residual && !h->d_user_R) DG_TRY(cudaMalloc(&h->d_user_R, ubytes));
  if (!h->stream) DG_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  return MC_OK;
}
}  // namespace

MC_API int mc_dg_ssprk3_user_host(mc_dg* h, double* U_host, double dt, int n_steps) {
  if (!h || !U_host) return mc_fail(MC_EINVAL, "null argument");
  if (h->ng) return mc_fail(MC_EINVAL, "partitioned operator: use the device entry points");
  if (int rc = user_staging(h, false)) return rc;
  const int64_t nblk = h->ne + h->ng;
  const size_t ubytes = sizeof(double) * size_t(h->n_user_rows) * h->ops->neq * h->ops->np;
  double* Ud = reinterpret_cast<double*>(h->d_host_U);
  DG_TRY(cudaMemcpyAsync(h->d_user, U_host, ubytes, cudaMemcpyHostToDevice, h->stream));
  if (int rc = mc_dg_user_to_internal(h, h->d_user, Ud, h->stream)) return rc;
  if (int rc = mc_dg_ssprk3(h, Ud, at_blocks(Ud, h, nblk), dt, n_steps, h->stream)) return rc;
  if (int rc = mc_dg_internal_to_user(h, Ud, h->d_user, h->stream)) return rc;
  DG_TRY(cudaMemcpyAsync(U_host, h->d_user, ubytes, cudaMemcpyDeviceToHost, h->stream));
  DG_TRY(cudaStreamSynchronize(h->stream));
  return MC_OK;
}

MC_API int mc_dg_rhs_user_host(mc_dg* h, const double* U_host, double* R_host, int strategy) {
  if (!h || !U_host || !R_host) return mc_fail(MC_EINVAL, "null argument");
  if (h->ng) return mc_fail(MC_EINVAL, "partitioned operator: use the device entry points");
  if (int rc = user_staging(h, true)) return rc;
  const int64_t nblk = h->ne + h->ng;
  const size_t ubytes = sizeof(double) * size_t(h->n_user_rows) * h->ops->neq * h->ops->np;
  double* Ud = reinterpret_cast<double*>(h->d_host_U);
  DG_TRY(cudaMemcpyAsync(h->d_user, U_host, ubytes, cudaMemcpyHostToDevice, h->stream));
  if (int rc = mc_dg_user_to_internal(h, h->d_user, Ud, h->stream)) return rc;
  if (int rc = mc_dg_rhs(h, Ud, at_blocks(Ud, h, 2 * nblk), strategy, h->stream)) return rc;
  DG_TRY(cudaMemsetAsync(h->d_user_R, 0, ubytes, h->stream));
  if (int rc = mc_dg_internal_to_user(h, at_blocks(Ud, h, 2 * nblk), h->d_user_R, h->stream))
    return rc;
  DG_TRY(cudaMemcpyAsync(R_host, h->d_user_R, ubytes, cudaMemcpyDeviceToHost, h->stream));
  DG_TRY(cudaStreamSynchronize(h->stream));
  return MC_OK;
}

}  // extern "C"
