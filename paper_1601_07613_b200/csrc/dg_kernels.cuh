// DG surface-integral kernels for sm_100a (fp64), templated on element
// kind, physics and polynomial degree.
//
// Algorithm 1 with Eq. (2): for each
// color, every surface evaluates the traces of its two elements at the
// surface quadrature points, the Lax-Friedrichs flux, and scatters
// -/+ s * sum_g w_g phi_j(g) Fhat_g straight into the residual blocks of its
// left / right element.  A valid coloring guarantees no element is touched
// twice in one launch, so the scatter is a plain read-modify-write:
// no atomics, no per-surface buffer.
//
// Thread mapping (the "surface group"): 2*NEQ lanes per surface, lane =
// (side, equation).  Each lane owns the N_p coefficients of ONE equation
// of ONE element in registers, computes its own trace component, and
// exchanges traces through warp shuffles so every lane can evaluate the
// (nonlinear) flux; the projection onto the basis is again per lane.
// Element blocks are [eq][j] contiguous doubles, so a lane's coefficients
// are one contiguous run (double2 loads when N_p*8 is a multiple of 16).
//
// Fusion: the volume integral of an element is
// computed in the pass where the element is first touched (its residual
// block is then written, never read) and, in an RK stage, the update
// U <- a*U0 + b*(U + dt*R) is applied in the pass where it is last
// touched (the residual block is then read but never written).  The
// update is in place: in that pass no other surface reads U_e.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/meshchroma_b200.h"

namespace mcdg {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;

enum Kind { TRI = 0, QUAD = 1, TET = 2 };
enum Phys { ADV = 0, EULER = 1 };

template <int K, int PH, int P>
struct Cfg {
  static constexpr int DIM = (K == TET) ? 3 : 2;
  static constexpr int NEQ = (PH == ADV) ? 1 : DIM + 2;
  static constexpr int NP = (K == TRI) ? (P + 1) * (P + 2) / 2
                          : (K == QUAD) ? (P + 1) * (P + 1)
                                        : (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NQF = (K == TET) ? (P + 1) * (P + 1) : P + 1;
  static constexpr int NQV = (K == TET) ? (P + 1) * (P + 1) * (P + 1) : (P + 1) * (P + 1);
  static constexpr int NCODES = (K == QUAD || K == TET) ? 24 : 18;
  static constexpr int G = 2 * NEQ;           // lanes per surface
  static constexpr int SPW = 32 / G;          // surfaces per warp
  static constexpr int GEOM = DIM + 2;        // doubles per surface geometry
  // packed table offsets (doubles): face_phi | face_w | vol_phi | vol_dphi | vol_w
  static constexpr int T_FPHI = 0;
  static constexpr int T_FW = T_FPHI + NCODES * NQF * NP;
  static constexpr int T_VPHI = T_FW + NQF;
  static constexpr int T_VDPHI = T_VPHI + NQV * NP;
  static constexpr int T_VW = T_VDPHI + DIM * NQV * NP;
  static constexpr int T_SIZE = T_VW + NQV;
};

struct Params {
  double gamma;
  double vel[3];
  double ff[5];
};

// Everything a kernel needs, passed by value.
struct View {
  const int32_t* left;
  const int32_t* right;
  const uint32_t* code;
  const double* geom;
  const double* jinv;
  const double* tables;
  const int64_t* slot_ptr;
  const int32_t* slots;
  int64_t n_elements;
  int64_t n_surfaces;
  int64_t stride;      // doubles per element block
  Params prm;
};

struct RK {
  double* U0;     // stage base state (read when a != 0; written when save_u0)
  double a, b, dt;
  int save_u0;    // first SSP-RK stage: U0 := U before the in-place update
};

// ------------------------------------------------------------- helpers
template <int N>
__device__ __forceinline__ void load_run(const double* __restrict__ src, double (&dst)[N]) {
  if constexpr ((N % 2) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      double2 v = __ldg(s2 + j);
      dst[2 * j] = v.x;
      dst[2 * j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) dst[j] = __ldg(src + j);
  }
}

// plain (non-__ldg) load for data written earlier in the same stream by
// other launches (residual partial sums)
template <int N>
__device__ __forceinline__ void load_rw(const double* src, double (&dst)[N]) {
  if constexpr ((N % 2) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      double2 v = s2[j];
      dst[2 * j] = v.x;
      dst[2 * j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) dst[j] = src[j];
  }
}

template <int N>
__device__ __forceinline__ void store_run(double* dst, const double (&src)[N]) {
  if constexpr ((N % 2) == 0) {
    double2* d2 = reinterpret_cast<double2*>(dst);
#pragma unroll
    for (int j = 0; j < N / 2; ++j) d2[j] = make_double2(src[2 * j], src[2 * j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) dst[j] = src[j];
  }
}

template <int DIM>
__device__ __forceinline__ double sel3(int i, double a, double b, double c) {
  return i == 0 ? a : (i == 1 ? b : c);
}

// ----------------------------------------------------------- physics
// Normal flux component `eq` of the Lax-Friedrichs flux.  sL/sR hold the
// full states (NEQ values) at one point; own values need no dynamic
// indexing: the caller passes this lane's components qL = sL[eq], qR.
template <int PH, int DIM, int NEQ>
struct Flux;

template <int DIM, int NEQ>
struct Flux<ADV, DIM, NEQ> {
  __device__ static __forceinline__ double numerical(const double*, const double*, double qL,
                                                     double qR, const double* n, int,
                                                     const Params& P) {
    double an = P.vel[0] * n[0] + P.vel[1] * n[1];
    if (DIM == 3) an += P.vel[2] * n[2];
    return 0.5 * an * (qL + qR) - 0.5 * fabs(an) * (qR - qL);
  }
  // contravariant volume flux Ft_r = sum_d Jinv[r][d] F_d for own component
  __device__ static __forceinline__ void volume(const double*, double q, const double* jinv,
                                                int, const Params& P, double* Ft) {
#pragma unroll
    for (int r = 0; r < DIM; ++r) {
      double a = jinv[r * DIM + 0] * P.vel[0] + jinv[r * DIM + 1] * P.vel[1];
      if (DIM == 3) a += jinv[r * DIM + 2] * P.vel[2];
      Ft[r] = a * q;
    }
  }
};

template <int DIM, int NEQ>
struct Flux<EULER, DIM, NEQ> {
  __device__ static __forceinline__ void prim(const double* s, const Params& P, double* u,
                                              double& p) {
    const double inv = 1.0 / s[0];
    double ke = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      u[d] = s[1 + d] * inv;
      ke += s[1 + d] * u[d];
    }
    p = (P.gamma - 1.0) * (s[NEQ - 1] - 0.5 * ke);
  }

  __device__ static __forceinline__ double numerical(const double* sL, const double* sR,
                                                     double qL, double qR, const double* n,
                                                     int eq, const Params& P) {
    double uL[DIM], uR[DIM], pL, pR;
    prim(sL, P, uL, pL);
    prim(sR, P, uR, pR);
    double vnL = 0.0, vnR = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      vnL += uL[d] * n[d];
      vnR += uR[d] * n[d];
    }
    const double cL = sqrt(P.gamma * pL / sL[0]);
    const double cR = sqrt(P.gamma * pR / sR[0]);
    const double lam = fmax(fabs(vnL) + cL, fabs(vnR) + cR);
    // F.n component: q*vn + p*m, m = 0 (mass), n_d (momentum d), vn (energy)
    double nm = 0.0;
    if (eq >= 1 && eq <= DIM) nm = sel3<DIM>(eq - 1, n[0], n[1], DIM == 3 ? n[2] : 0.0);
    const bool energy = eq == NEQ - 1;
    const double fL = qL * vnL + pL * (energy ? vnL : nm);
    const double fR = qR * vnR + pR * (energy ? vnR : nm);
    return 0.5 * (fL + fR) - 0.5 * lam * (qR - qL);
  }

  __device__ static __forceinline__ void volume(const double* s, double q, const double* jinv,
                                                int eq, const Params& P, double* Ft) {
    double u[DIM], p;
    prim(s, P, u, p);
    const bool energy = eq == NEQ - 1;
    const double coef = energy ? q + p : q;
#pragma unroll
    for (int r = 0; r < DIM; ++r) {
      double ut = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) ut += jinv[r * DIM + d] * u[d];
      double extra = 0.0;
      if (eq >= 1 && eq <= DIM)
        extra = p * sel3<DIM>(eq - 1, jinv[r * DIM + 0], jinv[r * DIM + 1],
                              DIM == 3 ? jinv[r * DIM + 2] : 0.0);
      Ft[r] = coef * ut + extra;
    }
  }
};

// ------------------------------------------------- table staging (smem)
template <class C>
__device__ __forceinline__ void stage_tables(const double* __restrict__ g, double* s) {
  for (int i = threadIdx.x; i < C::T_SIZE; i += blockDim.x) s[i] = __ldg(g + i);
  __syncthreads();
}

// Volume contribution of one element for this lane's equation, added into
// acc.  All lanes of the warp must call it (shuffles); `base` is the first
// lane of this lane's element group (NEQ lanes).
template <class C, int PH>
__device__ __forceinline__ void volume_into(const double* st, const double (&u)[C::NP],
                                            const double* jinv, int base, int eq,
                                            const Params& prm, double (&acc)[C::NP]) {
  const double* vphi = st + C::T_VPHI;
  const double* vdphi = st + C::T_VDPHI;
  const double* vw = st + C::T_VW;
#pragma unroll 1
  for (int q = 0; q < C::NQV; ++q) {
    double uq = 0.0;
#pragma unroll
    for (int j = 0; j < C::NP; ++j) uq = fma(vphi[q * C::NP + j], u[j], uq);
    double s[C::NEQ];
#pragma unroll
    for (int k = 0; k < C::NEQ; ++k) s[k] = __shfl_sync(kFull, uq, base + k);
    double Ft[C::DIM];
    Flux<PH, C::DIM, C::NEQ>::volume(s, uq, jinv, eq, prm, Ft);
    const double w = vw[q];
#pragma unroll
    for (int r = 0; r < C::DIM; ++r) Ft[r] *= w;
#pragma unroll
    for (int j = 0; j < C::NP; ++j) {
      double t = acc[j];
#pragma unroll
      for (int r = 0; r < C::DIM; ++r) t = fma(vdphi[(r * C::NQV + q) * C::NP + j], Ft[r], t);
      acc[j] = t;
    }
  }
}

// Surface contribution of one surface for this lane (side, eq) into acc.
template <class C, int PH>
__device__ __forceinline__ void surface_into(const double* st, const double (&u)[C::NP],
                                             bool has, bool boundary, int mycode, int side,
                                             int eq, int lane, int grp_base, const double* n,
                                             double scale, const Params& prm,
                                             double (&acc)[C::NP]) {
  const double* fphi = st + C::T_FPHI + mycode * (C::NQF * C::NP);
  const double* fw = st + C::T_FW;
  const double sign = side ? 1.0 : -1.0;
#pragma unroll 1
  for (int g = 0; g < C::NQF; ++g) {
    double tr = 0.0;
    if (has) {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) tr = fma(fphi[g * C::NP + j], u[j], tr);
    }
    double sL[C::NEQ], sR[C::NEQ];
#pragma unroll
    for (int k = 0; k < C::NEQ; ++k) {
      sL[k] = __shfl_sync(kFull, tr, grp_base + k);
      sR[k] = __shfl_sync(kFull, tr, grp_base + C::NEQ + k);
    }
    // partner value of this lane's own equation
    double qL = __shfl_sync(kFull, tr, grp_base + eq);
    double qR = __shfl_sync(kFull, tr, grp_base + C::NEQ + eq);
    if (boundary) {  // far-field ghost state
#pragma unroll
      for (int k = 0; k < C::NEQ; ++k) sR[k] = prm.ff[k];
      qR = prm.ff[eq];
    }
    const double fh = Flux<PH, C::DIM, C::NEQ>::numerical(sL, sR, qL, qR, n, eq, prm);
    const double coef = sign * scale * fw[g] * fh;
#pragma unroll
    for (int j = 0; j < C::NP; ++j) acc[j] = fma(coef, fphi[g * C::NP + j], acc[j]);
  }
}

struct Lane {
  int lane, grp, r, side, eq, grp_base, side_base;
  bool active;
};

template <class C>
__device__ __forceinline__ Lane lane_info() {
  Lane L;
  L.lane = threadIdx.x & 31;
  L.grp = L.lane / C::G;
  L.r = L.lane - L.grp * C::G;
  L.side = L.r / C::NEQ;
  L.eq = L.r - L.side * C::NEQ;
  L.active = L.grp < C::SPW;
  if (!L.active) {  // idle tail lanes shadow group 0 (results discarded)
    L.grp = 0;
  }
  L.grp_base = L.grp * C::G;
  L.side_base = L.grp_base + L.side * C::NEQ;
  return L;
}

// --------------------------------------------------------------- kernels
// One color: surfaces [begin, end) of the color-major list.
template <class C, int PH, bool kRK>
__global__ void __launch_bounds__(kThreads)
k_surface_colored(View v, double* __restrict__ U, double* __restrict__ R, RK rk, int64_t begin,
                  int64_t end) {
  extern __shared__ double st[];
  stage_tables<C>(v.tables, st);
  const Lane ln = lane_info<C>();
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t tile = begin + warp * C::SPW; tile < end; tile += nwarp * C::SPW) {
    const int64_t s = tile + ln.grp;
    const bool valid = ln.active && s < end;
    int L = 0, Rr = -1;
    uint32_t code = 0;
    double n[C::DIM];
    double scale = 0.0;
    if (s < end) {
      L = __ldg(v.left + s);
      Rr = __ldg(v.right + s);
      code = __ldg(v.code + s);
      const double* gm = v.geom + s * C::GEOM;
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) n[d] = __ldg(gm + d);
      scale = __ldg(gm + C::DIM + ln.side);
    } else {
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) n[d] = 0.0;
      n[0] = 1.0;
    }
    const bool boundary = Rr < 0;
    const int e = ln.side ? Rr : L;
    const bool ghost = ln.side && (code & MC_FLAG_R_GHOST);
    const bool has = valid && e >= 0;
    const bool owner = has && !ghost;
    const int mycode = ln.side ? int((code >> 6) & 63u) : int(code & 63u);
    const bool first = owner && (code & (ln.side ? MC_FLAG_R_FIRST : MC_FLAG_L_FIRST));
    const bool last = owner && (code & (ln.side ? MC_FLAG_R_LAST : MC_FLAG_L_LAST));

    double u[C::NP], acc[C::NP];
    const int64_t off = int64_t(has ? e : 0) * v.stride + ln.eq * C::NP;
    if (has) {
      load_run<C::NP>(U + off, u);
    } else {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) u[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
    if (__any_sync(kFull, first)) {
      double jinv[C::DIM * C::DIM];
      const double* jp = v.jinv + int64_t(has ? e : 0) * (C::DIM * C::DIM);
#pragma unroll
      for (int k = 0; k < C::DIM * C::DIM; ++k) jinv[k] = has ? __ldg(jp + k) : 0.0;
      volume_into<C, PH>(st, u, jinv, ln.side_base, ln.eq, v.prm, acc);
      if (!first) {
#pragma unroll
        for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
      }
    }
    if (owner && !first) load_rw<C::NP>(R + off, acc);
    surface_into<C, PH>(st, u, has, boundary, mycode, ln.side, ln.eq, ln.lane, ln.grp_base, n,
                        scale, v.prm, acc);
    if (owner) {
      if (kRK && last) {
        if (rk.save_u0) store_run<C::NP>(rk.U0 + off, u);
        if (rk.a != 0.0) {
          double u0[C::NP];
          load_run<C::NP>(rk.U0 + off, u0);
#pragma unroll
          for (int j = 0; j < C::NP; ++j) acc[j] = rk.a * u0[j] + rk.b * fma(rk.dt, acc[j], u[j]);
        } else {
#pragma unroll
          for (int j = 0; j < C::NP; ++j) acc[j] = rk.b * fma(rk.dt, acc[j], u[j]);
        }
        store_run<C::NP>(U + off, acc);
      } else {
        store_run<C::NP>(R + off, acc);
      }
    }
  }
}

// Volume integral for all owned elements: NEQ lanes per element.
template <class C, int PH>
__global__ void __launch_bounds__(kThreads)
k_volume(View v, const double* __restrict__ U, double* __restrict__ R) {
  extern __shared__ double st[];
  stage_tables<C>(v.tables, st);
  constexpr int EPW = 32 / C::NEQ;
  const int lane = threadIdx.x & 31;
  int grp = lane / C::NEQ;
  const int eq = lane - grp * C::NEQ;
  const bool act = grp < EPW;
  if (!act) grp = 0;
  const int base = grp * C::NEQ;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t tile = warp * EPW; tile < v.n_elements; tile += nwarp * EPW) {
    const int64_t e = tile + grp;
    const bool has = act && e < v.n_elements;
    const int64_t off = (has ? e : 0) * v.stride + eq * C::NP;
    double u[C::NP], acc[C::NP], jinv[C::DIM * C::DIM];
    if (has) load_run<C::NP>(U + off, u);
    else {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) u[j] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < C::DIM * C::DIM; ++k)
      jinv[k] = has ? __ldg(v.jinv + (has ? e : 0) * (C::DIM * C::DIM) + k) : 0.0;
#pragma unroll
    for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
    volume_into<C, PH>(st, u, jinv, base, eq, v.prm, acc);
    if (has) store_run<C::NP>(R + off, acc);
  }
}

// Surface contributions of ALL surfaces (no coloring) to either the
// 2*ns buffer (kAtomic = false: slot 2s+side) or atomically into R.
template <class C, int PH, bool kAtomic>
__global__ void __launch_bounds__(kThreads)
k_surface_uncolored(View v, const double* __restrict__ U, double* __restrict__ out) {
  extern __shared__ double st[];
  stage_tables<C>(v.tables, st);
  const Lane ln = lane_info<C>();
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t end = v.n_surfaces;
  for (int64_t tile = warp * C::SPW; tile < end; tile += nwarp * C::SPW) {
    const int64_t s = tile + ln.grp;
    const bool valid = ln.active && s < end;
    int L = 0, Rr = -1;
    uint32_t code = 0;
    double n[C::DIM];
    double scale = 0.0;
    if (s < end) {
      L = __ldg(v.left + s);
      Rr = __ldg(v.right + s);
      code = __ldg(v.code + s);
      const double* gm = v.geom + s * C::GEOM;
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) n[d] = __ldg(gm + d);
      scale = __ldg(gm + C::DIM + ln.side);
    } else {
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) n[d] = 0.0;
      n[0] = 1.0;
    }
    const bool boundary = Rr < 0;
    const int e = ln.side ? Rr : L;
    const bool ghost = ln.side && (code & MC_FLAG_R_GHOST);
    const bool has = valid && e >= 0;
    const bool owner = has && !ghost;
    const int mycode = ln.side ? int((code >> 6) & 63u) : int(code & 63u);
    double u[C::NP], acc[C::NP];
    if (has) load_run<C::NP>(U + int64_t(e) * v.stride + ln.eq * C::NP, u);
    else {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) u[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
    surface_into<C, PH>(st, u, has, boundary, mycode, ln.side, ln.eq, ln.lane, ln.grp_base, n,
                        scale, v.prm, acc);
    if (kAtomic) {
      if (owner) {
        double* dst = out + int64_t(e) * v.stride + ln.eq * C::NP;
#pragma unroll
        for (int j = 0; j < C::NP; ++j) atomicAdd(dst + j, acc[j]);
      }
    } else if (valid) {
      // buffer slot 2s+side holds this side's contribution (0 if absent)
      double* dst = out + (2 * s + ln.side) * v.stride + ln.eq * C::NP;
      if (!owner) {
#pragma unroll
        for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
      }
      store_run<C::NP>(dst, acc);
    }
  }
}

// Buffer-and-reduce phase two: R[e] += sum of its slots (local side order).
template <class C>
__global__ void __launch_bounds__(kThreads)
k_gather(View v, const double* __restrict__ buf, double* __restrict__ R) {
  constexpr int W = C::NEQ * C::NP;
  const int64_t total = v.n_elements * W;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = i / W;
    const int64_t k = i - e * W;
    double acc = R[e * v.stride + k];
    const int64_t b = __ldg(v.slot_ptr + e), f = __ldg(v.slot_ptr + e + 1);
    for (int64_t t = b; t < f; ++t) acc += __ldg(buf + int64_t(__ldg(v.slots + t)) * v.stride + k);
    R[e * v.stride + k] = acc;
  }
}

// U <- a*U0 + b*(U + dt*R) over owned blocks (unfused strategies).
static __global__ void __launch_bounds__(kThreads)
k_rk_update(int64_t n, double* __restrict__ U, const double* __restrict__ U0,
            const double* __restrict__ R, double a, double b, double dt) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    U[i] = a * U0[i] + b * fma(dt, R[i], U[i]);
}

}  // namespace mcdg
