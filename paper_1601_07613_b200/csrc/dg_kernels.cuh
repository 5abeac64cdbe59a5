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
// Warp organisation ("surface group"): 2*NEQ lanes per surface, lane =
// (side, equation).  A lane owns the N_p coefficients of ONE equation of
// ONE element in registers: it loads them (one contiguous run, [eq][j]
// element blocks, 16-byte vector loads), evaluates its own trace
// components, and finally projects the fluxes back onto its basis and
// stores.  The nonlinear flux in between needs the full state at a point,
// so each flux is evaluated exactly ONCE per quadrature point as a warp
// "task": traces are staged in a per-warp shared-memory scratch, the
// warp's 32 lanes split the (surface, point) and (element, volume point)
// tasks among themselves, and the results come back through the scratch.
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

// HYB: conforming triangle + quad mix; quad-sized blocks (triangles use the
// first (p+1)(p+2)/2 modes of each equation), 24 quad + 18 triangle face
// codes, the volume tables hold the quad rule's rows then the triangle's
enum Kind { TRI = 0, QUAD = 1, TET = 2, HYB = 3 };
enum Phys { ADV = 0, EULER = 1 };

template <int K, int PH, int P>
struct Cfg {
  static constexpr int KIND = K, PDEG = P;
  static constexpr int DIM = (K == TET) ? 3 : 2;
  static constexpr int NEQ = (PH == ADV) ? 1 : DIM + 2;
  static constexpr int NP = (K == TRI) ? (P + 1) * (P + 2) / 2
                          : (K == QUAD || K == HYB) ? (P + 1) * (P + 1)
                                                    : (P + 1) * (P + 2) * (P + 3) / 6;
  // quadrature (dg/basis.py): degree-5 symmetric rules for p = 2 on simplices
  static constexpr int NQF = (K == TET) ? (P == 2 ? 7 : (P + 1) * (P + 1)) : P + 1;
  static constexpr int NQV_TRI = (P == 2) ? 7 : (P + 1) * (P + 1);
  static constexpr int NQV_QUAD = (P + 1) * (P + 1);   // HYB: quad rows [0, NQV_QUAD)
  static constexpr int NQV = (K == TET) ? (P == 2 ? 14 : (P + 1) * (P + 1) * (P + 1))
                           : (K == TRI) ? NQV_TRI
                           : (K == HYB) ? NQV_QUAD + NQV_TRI : NQV_QUAD;
  static constexpr int NCODES = (K == QUAD || K == TET) ? 24 : (K == HYB) ? 42 : 18;
  static constexpr int TRI_CODE0 = 24;                  // HYB: first triangle face code
#ifdef MC_DG_DMMA
  static constexpr bool DMMA_ON = (K != TET);
#else
  static constexpr bool DMMA_ON = false;
#endif
  static constexpr int G = 2 * NEQ;           // lanes per surface
  static constexpr int SPW = 32 / G;          // surfaces per warp
  static constexpr int ES = 2 * SPW;          // element slots per warp (surface kernels)
  static constexpr int GEOM = DIM + 2;        // doubles per surface geometry
  // volume points per task chunk: about one task per lane per chunk
  static constexpr int QC = (32 / ES) < 1 ? 1 : ((32 / ES) > NQV ? NQV : (32 / ES));
  // block shape: tets carry large tables, use smaller blocks
  static constexpr int WARPS = (K == TET) ? 4 : 8;
  static constexpr int THREADS = 32 * WARPS;
#ifndef MC_MINB_2D
#define MC_MINB_2D 3
#endif
#ifndef MC_MINB_3D
#define MC_MINB_3D 4
#endif
  static constexpr int MINB = (K == TET) ? MC_MINB_3D : MC_MINB_2D;
  // packed table offsets (doubles): face_phi | face_w | vol_phi | vol_dphi | vol_w
  static constexpr int T_FPHI = 0;
  static constexpr int T_FW = T_FPHI + NCODES * NQF * NP;
  static constexpr int T_VPHI = T_FW + NQF;
  static constexpr int T_VDPHI = T_VPHI + NQV * NP;
  static constexpr int T_VW = T_VDPHI + DIM * NQV * NP;
  // Projection through P_{p-1} (simplices, register kernels): the reference
  // gradients of the P_p modes lie in P_{p-1} (NPL modes), so
  //   sum_q w_q dphi_r[q][j] G[q] = sum_m D_r[j][m] (sum_q w_q phi_m[q] G[q]).
  // Tables (computed at operator creation from vol_phi / vol_dphi):
  // WPSI[q][m] = w_q phi_m(q), DMAT[r][j][m]; modes are ordered by total
  // degree, so D_r[j][m] = 0 unless m < NPL(deg(j) - 1).
  static constexpr int NPL = (K == QUAD || K == HYB || NEQ * NP > 64) ? 1
                           : (K == TRI) ? P * (P + 1) / 2 : P * (P + 1) * (P + 2) / 6;
#ifdef MC_NO_P1PROJ
  static constexpr bool P1PROJ = false;
#else
  static constexpr bool P1PROJ = (K != QUAD && K != HYB) && P >= 1 && NEQ * NP <= 64;
#endif
  static constexpr int T_WPSI = T_VW + NQV;
  static constexpr int T_DMAT = T_WPSI + NQV * NPL;
  static constexpr int T_SIZE = T_DMAT + DIM * NP * NPL;
  // shared-memory copy: rows padded to an even length so that pairs of
  // basis values are one 16-byte broadcast load (LDS.128)
  static constexpr int NPP = (NP + 1) & ~1;
  static constexpr int S_FPHI = 0;
  static constexpr int S_FW = S_FPHI + NCODES * NQF * NPP;
  static constexpr int S_VPHI = S_FW + ((NQF + 1) & ~1);
  static constexpr int S_VDPHI = S_VPHI + NQV * NPP;
  static constexpr int S_VW = S_VDPHI + DIM * NQV * NPP;
  static constexpr int S_WPSI = S_VW + ((NQV + 1) & ~1);
  static constexpr int S_DMAT = S_WPSI + ((NQV * NPL + 1) & ~1);
  static constexpr int S_SIZE = S_DMAT + ((DIM * NP * NPL + 1) & ~1);
  // per-warp scratch (doubles) for the surface kernels.  Every array is
  // indexed so that the lane-parallel accesses (one lane per task or per
  // (slot, eq)) step by an ODD number of doubles: conflict-free banks.
  static constexpr int SV = NEQ | 1;                              // padded state stride
  static constexpr int JIS = (DIM * DIM) | 1;                     // padded Jinv stride
  static constexpr int W_TR = 0;                                  // [2][NQF][SPW][SV]
  static constexpr int W_FS = W_TR + 2 * NQF * SPW * SV;          // [NQF][SPW][SV]
  // the DMMA volume scratch {RM, VQ, FT} aliases TR/FS (used only later)
  static constexpr int W_UNION = DMMA_ON
      ? (8 * ((NP + 7) / 8) * 32 + 8 * 32 + 4 * DIM * 36) : 0;
  static constexpr int W_FS_END = W_FS + NQF * SPW * SV;
  static constexpr int W_NRM = ((W_FS_END > W_UNION ? W_FS_END : W_UNION) + 1) & ~1;  // [SPW][DIM]
  static constexpr int W_JI = W_NRM + SPW * DIM;                  // [ES][JIS]
  static constexpr bool VTASK = !DMMA_ON;                          // task volume path
  static constexpr int W_VS = W_JI + ES * JIS;                    // [QC][ES][SV]
  static constexpr int W_VF = W_VS + (VTASK ? QC * ES * SV : 0);  // [DIM][QC][ES][SV]
  static constexpr int W_FLAG = W_VF + (VTASK ? DIM * QC * ES * SV : 0);  // ints: valid, need
  static constexpr int W_SIZE_T = (W_FLAG + (SPW + ES + 1) / 2 + 2) & ~1;
  // ---- FP64 tensor-core (DMMA m8n8k4) volume integral, 2D kinds -------
  // trace  V[q][col] = sum_j Phi[q][j] C[j][col]         (MT x KT tiles)
  // project R[j][col] = sum_kk Dt[j][kk] Ft[kk][col], kk = q*DIM + r
  // col = element slot * NEQ + eq = lane id (32 columns = 4 N tiles)
#ifdef MC_DG_DMMA
  static constexpr bool DMMA = (K != TET) && (ES * NEQ == 32);
#else
  // measured slower than the task path on B200: fragment traffic makes the
  // kernel shared-memory bound (profiles/)
  static constexpr bool DMMA = false;
#endif
  static constexpr int MT = (NQV + 7) / 8;       // 8-point chunks / trace M tiles
  static constexpr int KT = (NP + 3) / 4;        // trace k steps
  static constexpr int MJ = (NP + 7) / 8;        // projection M tiles
  static constexpr int KS = MT * 2 * DIM;        // projection k steps (4 kk rows each)
  static constexpr int LDB = 36;                 // padded row stride of B tiles
  static constexpr int S_AFP = S_SIZE;                     // [MT][KT][32] A fragments
  static constexpr int S_AFD = S_AFP + MT * KT * 32;       // [MJ][KS][32]
  static constexpr int S_TOTAL = ((DMMA ? S_AFD + MJ * KS * 32 : S_SIZE) + 1) & ~1;
  static constexpr int D_RM = 0;                                  // [8*MJ][32]
  static constexpr int D_VQ = D_RM + 8 * MJ * 32;                 // [8][32]
  static constexpr int D_FT = D_VQ + 8 * 32;                      // [4*DIM][32]
  static constexpr int D_END = D_FT + 4 * DIM * 32;
  static constexpr int D_CM = W_SIZE_T;                           // [4*KT][LDB], persists
  static constexpr int W_SIZE = DMMA ? (D_CM + 4 * KT * LDB) : W_SIZE_T;  // even: 16-B aligned
  static_assert(W_SIZE % 2 == 0 && S_TOTAL % 2 == 0 && W_NRM % 2 == 0, "16-byte alignment");
  static_assert(!DMMA || D_END <= W_NRM, "DMMA scratch must fit in the aliased region");
  static constexpr int SMEM = (S_TOTAL + WARPS * W_SIZE) * 8;
  // element-major volume kernel: NEQ lanes per element
  static constexpr int EPW = 32 / NEQ;
  static constexpr int QCV = (32 / EPW) < 1 ? 1 : ((32 / EPW) > NQV ? NQV : (32 / EPW));
  static constexpr int V_JI = 0;
  static constexpr int V_VS = V_JI + EPW * JIS;
  static constexpr int V_VF = V_VS + EPW * QCV * SV;
  static constexpr int V_FLAG = V_VF + EPW * QCV * DIM * SV;
  static constexpr int V_SIZE = V_FLAG + (EPW + 1) / 2 + 1;
  static constexpr int VSMEM = (S_TOTAL + WARPS * V_SIZE) * 8;
};

// Volume tables (basis values, reference gradients, weights at the volume
// points) in constant memory, same padded layout as the shared-memory copy
// from S_VPHI on.  Every lane of a warp reads the same entry at the same
// time (uniform index), so these become uniform-datapath loads (LDCU) that
// cost no shared-memory wavefronts.  One array per configuration; filled by
// Instance::upload_const at operator creation.  Used by the register
// kernels (c2: 3.43 -> 3.53 G edges/s, c3: 0.94 -> 0.97 with warp-uniform
// control flow around the reads); the group kernel keeps the shared-memory
// copy (from constant memory c4 drops 0.92 -> 0.81, even with uniform
// loops).  MC_SMEM_VOLTAB forces shared memory.
template <int K, int P>
__constant__ double c_voltab[Cfg<K, ADV, P>::S_SIZE - Cfg<K, ADV, P>::S_VPHI];

template <class C, bool kConst>
__device__ __forceinline__ const double* vol_tables(const double* st) {
#ifdef MC_SMEM_VOLTAB
  constexpr bool use = false;
#else
  constexpr bool use = kConst;
#endif
  if constexpr (use) {
    (void)st;
    return c_voltab<C::KIND, C::PDEG>;
  } else {
    return st + C::S_VPHI;
  }
}

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
  const double* ptables;   // padded shared-memory layout, in global memory (L1-cached reads)
  const int64_t* slot_ptr;
  const int32_t* slots;
  int64_t n_elements;
  int64_t n_surfaces;
  int64_t stride;      // doubles per element block
  Params prm;
  const uint8_t* ekind;     // HYB: per element 0 = triangle, 1 = quad
  // partitioned runs: the last-touch pass of an RK stage also writes each
  // interface element's new block into its slot of the ghost-exchange send
  // buffer (send_slot[e] >= 0), so the next stage posts it without a pack
  const int32_t* send_slot;
  void* send_buf;          // element blocks of the state type (double / float)
  // peer-push exchange (mc_dg_set_push_rows): the last-touch pass also
  // stores every interface element's new block straight into its rows in
  // the peers' state arrays (NVLink P2P stores through mapped peer memory),
  // push_dst[push_ptr[e] .. push_ptr[e+1]) byte addresses, + push_shift
  // state values (the ghost copy the peers read next stage).  ghost_par
  // >= 0: ghost rows are double-buffered (ghost g at rows ne + 2g + parity)
  // and this launch reads parity ghost_par
  const int64_t* push_ptr;
  const unsigned long long* push_dst;
  int64_t push_shift;
  int ghost_par;
};

struct RK {
  void* U0;       // stage base state (read when a != 0; written when save_u0), state type
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

// plain (coherent) load for residual partial sums written by earlier launches
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

// sum_j row[j] * u[j] with 16-byte loads of the (even-padded) table row
template <int N>
__device__ __forceinline__ double dot_row(const double* row, const double (&u)[N]) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const double2 a = r2[j];
    t = fma(a.x, u[2 * j], t);
    t = fma(a.y, u[2 * j + 1], t);
  }
  if constexpr (N % 2) t = fma(row[N - 1], u[N - 1], t);
  return t;
}

// acc[j] += f * row[j]
template <int N>
__device__ __forceinline__ void axpy_row(const double* row, double f, double (&acc)[N]) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const double2 a = r2[j];
    acc[2 * j] = fma(a.x, f, acc[2 * j]);
    acc[2 * j + 1] = fma(a.y, f, acc[2 * j + 1]);
  }
  if constexpr (N % 2) acc[N - 1] = fma(row[N - 1], f, acc[N - 1]);
}

// ----------------------------------------------------------- physics
// Full-state flux evaluations, one call per quadrature point (a "task").
template <int PH, int DIM, int NEQ>
struct Physics;

template <int DIM, int NEQ>
struct Physics<ADV, DIM, NEQ> {
  // Fhat . n (upwind = Lax-Friedrichs with lambda = |a.n|)
  template <bool kFast = true>
  __device__ static __forceinline__ void lf(const double* sL, const double* sR, const double* n,
                                            const Params& P, double* out) {
    double an = P.vel[0] * n[0] + P.vel[1] * n[1];
    if (DIM == 3) an += P.vel[2] * n[2];
    out[0] = 0.5 * an * (sL[0] + sR[0]) - 0.5 * fabs(an) * (sR[0] - sL[0]);
  }
  // contravariant flux Ft[r][k] = sum_d Jinv[r][d] F_d(s)[k]
  template <bool kFast = true>
  __device__ static __forceinline__ void vflux(const double* s, const double* ji,
                                               const Params& P, double* Ft) {
#pragma unroll
    for (int r = 0; r < DIM; ++r) {
      double a = ji[r * DIM + 0] * P.vel[0] + ji[r * DIM + 1] * P.vel[1];
      if (DIM == 3) a += ji[r * DIM + 2] * P.vel[2];
      Ft[r] = a * s[0];
    }
  }
  // physical flux F[d][k] (the Jacobian is applied later, per element)
  __device__ static __forceinline__ void pflux(const double* s, const Params& P, double* F) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) F[d] = P.vel[d] * s[0];
  }
};

// fp64 reciprocal and square root for the flux: the hardware approximation
// (MUFU.RCP64H / MUFU.RSQ64H) refined by Newton steps to full double
// precision (within an ulp or two of the IEEE result), without the
// special-case slow path of the IEEE division / square root.  Densities and
// pressures are positive and normal here; MC_IEEE_DIV restores the IEEE
// operations.
#ifdef MC_IEEE_DIV
constexpr bool kFluxFastMath = false;
#else
constexpr bool kFluxFastMath = true;
#endif

template <bool kFast = true>
__device__ __forceinline__ double flux_rcp(double x) {
  if constexpr (!(kFast && kFluxFastMath)) {
    return 1.0 / x;
  } else {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
  }
}

template <bool kFast = true>
__device__ __forceinline__ double flux_sqrt(double x) {
  if constexpr (!(kFast && kFluxFastMath)) {
    return sqrt(x);
  } else {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    // y <- y (3 - x y^2) / 2, twice; then sqrt = x y with one Heron correction
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    const double s0 = x * y;
    return fma(fma(-s0, s0, x), 0.5 * y, s0);
  }
}

template <int DIM, int NEQ>
struct Physics<EULER, DIM, NEQ> {
  // kFast: Newton-refined MUFU reciprocal / square root.  Measured: wins in
  // the register kernels (c2 +1 %, c3 +2 %, c4 +3 %), loses in the group
  // kernel (-5 %, register pressure), which passes false.
  template <bool kFast = true>
  __device__ static __forceinline__ void prim(const double* s, const Params& P, double* u,
                                              double& p, double& inv) {
    inv = flux_rcp<kFast>(s[0]);
    double ke = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      u[d] = s[1 + d] * inv;
      ke += s[1 + d] * u[d];
    }
    p = (P.gamma - 1.0) * (s[NEQ - 1] - 0.5 * ke);
  }

  template <bool kFast = true>
  __device__ static __forceinline__ void lf(const double* sL, const double* sR, const double* n,
                                            const Params& P, double* out) {
    double uL[DIM], uR[DIM], pL, pR, iL, iR;
    prim<kFast>(sL, P, uL, pL, iL);
    prim<kFast>(sR, P, uR, pR, iR);
    double vnL = 0.0, vnR = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      vnL += uL[d] * n[d];
      vnR += uR[d] * n[d];
    }
    // sound speeds from the reciprocal density prim() already formed (one
    // fp64 division per state instead of two)
    const double cL = flux_sqrt<kFast>(P.gamma * pL * iL);
    const double cR = flux_sqrt<kFast>(P.gamma * pR * iR);
    const double lam = fmax(fabs(vnL) + cL, fabs(vnR) + cR);
    // F.n = s*vn + p*(0, n, vn)
    out[0] = 0.5 * (sL[0] * vnL + sR[0] * vnR) - 0.5 * lam * (sR[0] - sL[0]);
#pragma unroll
    for (int d = 0; d < DIM; ++d)
      out[1 + d] = 0.5 * ((sL[1 + d] * vnL + pL * n[d]) + (sR[1 + d] * vnR + pR * n[d])) -
                   0.5 * lam * (sR[1 + d] - sL[1 + d]);
    out[NEQ - 1] = 0.5 * ((sL[NEQ - 1] + pL) * vnL + (sR[NEQ - 1] + pR) * vnR) -
                   0.5 * lam * (sR[NEQ - 1] - sL[NEQ - 1]);
  }

  // physical flux F[d][k]: (m_d, m u_d + p e_d, (E + p) u_d)
  __device__ static __forceinline__ void pflux(const double* s, const Params& P, double* F) {
    double u[DIM], p, inv;
    prim<true>(s, P, u, p, inv);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      F[d * NEQ + 0] = s[1 + d];
#pragma unroll
      for (int e = 0; e < DIM; ++e) F[d * NEQ + 1 + e] = s[1 + e] * u[d] + (e == d ? p : 0.0);
      F[d * NEQ + NEQ - 1] = (s[NEQ - 1] + p) * u[d];
    }
  }

  template <bool kFast = true>
  __device__ static __forceinline__ void vflux(const double* s, const double* ji,
                                               const Params& P, double* Ft) {
    double u[DIM], p, inv;
    prim<kFast>(s, P, u, p, inv);
#pragma unroll
    for (int r = 0; r < DIM; ++r) {
      double ut = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) ut += ji[r * DIM + d] * u[d];
      Ft[r * NEQ + 0] = s[0] * ut;
#pragma unroll
      for (int d = 0; d < DIM; ++d) Ft[r * NEQ + 1 + d] = s[1 + d] * ut + p * ji[r * DIM + d];
      Ft[r * NEQ + NEQ - 1] = (s[NEQ - 1] + p) * ut;
    }
  }
};

// ------------------------------------------------- table staging (smem)
template <class C>
__device__ __forceinline__ void stage_tables(const double* __restrict__ g, double* s) {
  // compact global layout -> padded shared layout
  for (int i = threadIdx.x; i < C::S_SIZE; i += blockDim.x) {
    double v = 0.0;
    if (i < C::S_FW) {
      const int row = i / C::NPP, j = i - row * C::NPP;
      if (j < C::NP) v = __ldg(g + C::T_FPHI + row * C::NP + j);
    } else if (i < C::S_VPHI) {
      const int k = i - C::S_FW;
      if (k < C::NQF) v = __ldg(g + C::T_FW + k);
    } else if (i < C::S_VW) {
      const int row = (i - C::S_VPHI) / C::NPP, j = (i - C::S_VPHI) - row * C::NPP;
      if (j < C::NP) v = __ldg(g + C::T_VPHI + row * C::NP + j);  // vphi and vdphi rows
    } else if (i < C::S_WPSI) {
      const int k = i - C::S_VW;
      if (k < C::NQV) v = __ldg(g + C::T_VW + k);
    } else if (i < C::S_DMAT) {
      const int k = i - C::S_WPSI;
      if (k < C::NQV * C::NPL) v = __ldg(g + C::T_WPSI + k);
    } else {
      const int k = i - C::S_DMAT;
      if (k < C::DIM * C::NP * C::NPL) v = __ldg(g + C::T_DMAT + k);
    }
    s[i] = v;
  }
  if constexpr (C::DMMA) {
    __syncthreads();
    // A fragments (row = lane >> 2, k = lane & 3) of Phi and of Dt
    for (int i = threadIdx.x; i < C::MT * C::KT * 32; i += blockDim.x) {
      const int l = i & 31, mk = i >> 5, m = mk / C::KT, k = mk - m * C::KT;
      const int q = 8 * m + (l >> 2), j = 4 * k + (l & 3);
      s[C::S_AFP + i] = (q < C::NQV && j < C::NP) ? s[C::S_VPHI + q * C::NPP + j] : 0.0;
    }
    for (int i = threadIdx.x; i < C::MJ * C::KS * 32; i += blockDim.x) {
      const int l = i & 31, mk = i >> 5, mj = mk / C::KS, kst = mk - mj * C::KS;
      // k step kst covers dimension r = kst % DIM of the 4 points 4*(kst / DIM) + 0..3
      const int j = 8 * mj + (l >> 2), r = kst % C::DIM, q = 4 * (kst / C::DIM) + (l & 3);
      s[C::S_AFD + i] = (j < C::NP && q < C::NQV) ? s[C::S_VDPHI + (r * C::NQV + q) * C::NPP + j] : 0.0;
    }
  }
  __syncthreads();
}

// Volume integral of the warp's NS element slots, added into acc of the
// lanes whose slot needs it.  Warp-uniform control flow; `vs`, `vf`, `ji`,
// `need` live in the warp scratch; slot jinv/need were written earlier.
// Task t = (point qq, slot e) with e fastest, so task-parallel scratch
// accesses step by the odd stride SV (bank-conflict free).
template <class C, int PH, int NS, int QCH>
__device__ __forceinline__ void volume_tasks(const double* st, double* vs, double* vf,
                                             const double* ji, const int* need,
                                             const double (&u)[C::NP], int slot, int eq,
                                             bool mine, int lane, const Params& prm,
                                             double (&acc)[C::NP]) {
  // shared memory here: the lane-predicated task loops read the constant
  // copy slower (measured c4 0.82 vs 0.92 G edges/s)
  const double* vphi = vol_tables<C, false>(st);
  const double* vdphi = vphi + (C::S_VDPHI - C::S_VPHI);
  const double* vw = vphi + (C::S_VW - C::S_VPHI);
#pragma unroll 1
  for (int q0 = 0; q0 < C::NQV; q0 += QCH) {
    const int nq = (C::NQV - q0) < QCH ? (C::NQV - q0) : QCH;
    if (mine) {
      for (int qq = 0; qq < nq; ++qq)
        vs[(qq * NS + slot) * C::SV + eq] = dot_row<C::NP>(vphi + (q0 + qq) * C::NPP, u);
    }
    __syncwarp();
    for (int t = lane; t < NS * QCH; t += 32) {
      const int qq = t / NS, e = t - qq * NS;
      if (qq < nq && need[e]) {
        double s[C::NEQ], Ft[C::DIM * C::NEQ];
#pragma unroll
        for (int k = 0; k < C::NEQ; ++k) s[k] = vs[t * C::SV + k];
        Physics<PH, C::DIM, C::NEQ>::template vflux<false>(s, ji + e * C::JIS, prm, Ft);
        const double w = vw[q0 + qq];
#pragma unroll
        for (int r = 0; r < C::DIM; ++r) {
#pragma unroll
          for (int k = 0; k < C::NEQ; ++k)
            vf[(r * QCH * NS + t) * C::SV + k] = w * Ft[r * C::NEQ + k];
        }
      }
    }
    __syncwarp();
    if (mine) {
      for (int qq = 0; qq < nq; ++qq) {
#pragma unroll
        for (int r = 0; r < C::DIM; ++r) {
          const double f = vf[((r * QCH + qq) * NS + slot) * C::SV + eq];
          axpy_row<C::NP>(vdphi + (r * C::NQV + q0 + qq) * C::NPP, f, acc);
        }
      }
    }
    __syncwarp();
  }
}

// D(8x8) += A(8x4, row) * B(4x8, col), fp64 tensor core.  Fragments:
// a = A[lane>>2][lane&3], b = B[lane&3][lane>>2], (d0,d1) = D[lane>>2][2(lane&3)+{0,1}]
__device__ __forceinline__ void dmma(double a, double b, double& d0, double& d1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Volume integral through DMMA (all 32 lanes = 32 (slot, eq) columns).
// Per 8-point chunk: trace (DMMA) -> VQ; per half chunk of 4 points one
// flux task per (point, slot) -> FT; projection (DMMA) accumulates in RM.
// VQ / FT / RM rows are XOR-swizzled so that both the fragment accesses and
// the task accesses hit each bank pair at most twice (2 wavefronts).
__device__ __forceinline__ int swz8(int row) { return (row & 3) | ((row & 4) << 1); }
__device__ __forceinline__ int swzf(int row) {  // FT rows: (0, 1, 10, 11)[row & 3]
  return (row & 1) | ((row & 2) ? 10 : 0);
}

template <class C, int PH>
__device__ __forceinline__ void volume_dmma(const double* st, double* ws, const int* need,
                                            const double (&u)[C::NP], bool mine, int lane,
                                            const Params& prm, double (&acc)[C::NP]) {
  double* cm = ws + C::D_CM;
  double* rm = ws + C::D_RM;
  double* vq = ws + C::D_VQ;
  double* ft = ws + C::D_FT;
  const double* ji = ws + C::W_JI;
  const double* afp = st + C::S_AFP;
  const double* afd = st + C::S_AFD;
  const double* vw = st + C::S_VW;
  const int r4 = lane & 3, c8 = lane >> 2;
#pragma unroll
  for (int j = 0; j < C::NP; ++j) cm[j * C::LDB + lane] = u[j];
  __syncwarp();
#pragma unroll 1
  for (int m = 0; m < C::MT; ++m) {
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int k = 0; k < C::KT; ++k)
        dmma(afp[(m * C::KT + k) * 32 + lane], cm[(4 * k + r4) * C::LDB + 8 * n + c8], d0, d1);
      const int col = 8 * n + 2 * r4, g = swz8(c8);
      vq[c8 * 32 + (col ^ g)] = d0;
      vq[c8 * 32 + ((col + 1) ^ g)] = d1;
    }
    __syncwarp();
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if (8 * m + 4 * h >= C::NQV) break;           // warp-uniform
      for (int t = lane; t < 4 * C::ES; t += 32) {
        const int qq = t / C::ES, e = t - qq * C::ES;
        const int q = 8 * m + 4 * h + qq;
        double Ft[C::DIM * C::NEQ];
        if (q < C::NQV && need[e]) {
          double sv[C::NEQ];
          const int row = 4 * h + qq, g = swz8(row);
#pragma unroll
          for (int k = 0; k < C::NEQ; ++k) sv[k] = vq[row * 32 + ((e * C::NEQ + k) ^ g)];
          Physics<PH, C::DIM, C::NEQ>::template vflux<false>(sv, ji + e * C::JIS, prm, Ft);
          const double w = vw[q];
#pragma unroll
          for (int k = 0; k < C::DIM * C::NEQ; ++k) Ft[k] *= w;
        } else {
#pragma unroll
          for (int k = 0; k < C::DIM * C::NEQ; ++k) Ft[k] = 0.0;
        }
#pragma unroll
        for (int r = 0; r < C::DIM; ++r) {
          const int row = 4 * r + qq, g = swzf(row);
#pragma unroll
          for (int k = 0; k < C::NEQ; ++k) ft[row * 32 + ((e * C::NEQ + k) ^ g)] = Ft[r * C::NEQ + k];
        }
      }
      __syncwarp();
#pragma unroll
      for (int mj = 0; mj < C::MJ; ++mj) {
        const int row = 8 * mj + c8, g = swz8(c8);
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          const int col = 8 * n + 2 * r4;
          double c0 = 0.0, c1 = 0.0;
          if (m > 0 || h > 0) {
            c0 = rm[row * 32 + (col ^ g)];
            c1 = rm[row * 32 + ((col + 1) ^ g)];
          }
#pragma unroll
          for (int sl = 0; sl < C::DIM; ++sl)
            dmma(afd[(mj * C::KS + (2 * m + h) * C::DIM + sl) * 32 + lane],
                 ft[(4 * sl + r4) * 32 + ((8 * n + c8) ^ swzf(r4))], c0, c1);
          rm[row * 32 + (col ^ g)] = c0;
          rm[row * 32 + ((col + 1) ^ g)] = c1;
        }
      }
      __syncwarp();
    }
  }
  if (mine) {
#pragma unroll
    for (int j = 0; j < C::NP; ++j) acc[j] += rm[j * 32 + (lane ^ swz8(j & 7))];
  }
  __syncwarp();
}

struct Lane {
  int lane, grp, side, eq, slot;
  bool active;
};

template <class C>
__device__ __forceinline__ Lane lane_info() {
  Lane L;
  L.lane = threadIdx.x & 31;
  L.grp = L.lane / C::G;
  const int r = L.lane - L.grp * C::G;
  L.side = r / C::NEQ;
  L.eq = r - L.side * C::NEQ;
  L.active = L.grp < C::SPW;
  if (!L.active) L.grp = 0;   // idle tail lanes never write shared state
  L.slot = 2 * L.grp + L.side;
  return L;
}

// Per-surface part shared by the colored and uncolored kernels: metadata,
// traces into the scratch, one LF flux per (surface, point) task, and the
// lift of this lane's flux component into acc.
struct SurfCtx {
  int L, R, e, mycode;
  uint32_t code;
  double scale;
  bool valid, has, owner, boundary;
};

template <class C>
__device__ __forceinline__ SurfCtx load_surface(const View& v, const Lane& ln, int64_t s,
                                                int64_t end, double* ws) {
  SurfCtx c;
  c.valid = ln.active && s < end;
  c.L = 0;
  c.R = -1;
  c.code = 0;
  c.scale = 0.0;
  if (c.valid) {
    c.L = __ldg(v.left + s);
    c.R = __ldg(v.right + s);
    c.code = __ldg(v.code + s);
    const double* gm = v.geom + s * C::GEOM;
    c.scale = __ldg(gm + C::DIM + ln.side);
    if (ln.side == 0 && ln.eq == 0) {
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) ws[C::W_NRM + ln.grp * C::DIM + d] = __ldg(gm + d);
    }
  }
  c.boundary = c.R < 0;
  c.e = ln.side ? c.R : c.L;
  c.has = c.valid && c.e >= 0;
  c.owner = c.has && !(ln.side && (c.code & MC_FLAG_R_GHOST));
  c.mycode = ln.side ? int((c.code >> 6) & 63u) : int(c.code & 63u);
  return c;
}

template <class C, int PH>
__device__ __forceinline__ void surface_tasks(const double* st, double* ws, const Lane& ln,
                                              const SurfCtx& c, const double (&u)[C::NP],
                                              const Params& prm, double (&acc)[C::NP]) {
  const double* fphi = st + C::S_FPHI + c.mycode * (C::NQF * C::NPP);
  const double* fw = st + C::S_FW;
  int* valid = reinterpret_cast<int*>(ws + C::W_FLAG);
  if (ln.active && ln.side == 0 && ln.eq == 0)
    valid[ln.grp] = c.valid ? ((c.code & MC_FLAG_FLIPPED) ? 2 : 1) : 0;
  if (ln.active) {
#pragma unroll 1
    for (int g = 0; g < C::NQF; ++g) {
      double tr = 0.0;
      if (c.has) {
        tr = dot_row<C::NP>(fphi + g * C::NPP, u);
      } else if (c.valid && ln.side == 1) {
        tr = prm.ff[ln.eq];  // far-field ghost state on physical boundaries
      }
      ws[C::W_TR + ((ln.side * C::NQF + g) * C::SPW + ln.grp) * C::SV + ln.eq] = tr;
    }
  }
  __syncwarp();
  for (int t = ln.lane; t < C::SPW * C::NQF; t += 32) {
    const int g = t / C::SPW, gs = t - g * C::SPW;
    if (valid[gs]) {
      double sL[C::NEQ], sR[C::NEQ], n[C::DIM], out[C::NEQ];
#pragma unroll
      for (int k = 0; k < C::NEQ; ++k) {
        sL[k] = ws[C::W_TR + t * C::SV + k];
        sR[k] = ws[C::W_TR + (C::NQF * C::SPW + t) * C::SV + k];
      }
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) n[d] = ws[C::W_NRM + gs * C::DIM + d];
      // flipped by the partitioner: canonical orientation, one call site
      const bool flip = valid[gs] == 2;
      double cL[C::NEQ], cR[C::NEQ];
#pragma unroll
      for (int k = 0; k < C::NEQ; ++k) {
        cL[k] = flip ? sR[k] : sL[k];
        cR[k] = flip ? sL[k] : sR[k];
      }
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) n[d] = flip ? -n[d] : n[d];
      Physics<PH, C::DIM, C::NEQ>::template lf<false>(cL, cR, n, prm, out);
      const double w = flip ? -fw[g] : fw[g];
#pragma unroll
      for (int k = 0; k < C::NEQ; ++k) ws[C::W_FS + t * C::SV + k] = w * out[k];
    }
  }
  __syncwarp();
  if (c.owner) {
    const double sc = ln.side ? c.scale : -c.scale;
#pragma unroll 1
    for (int g = 0; g < C::NQF; ++g) {
      const double f = sc * ws[C::W_FS + (g * C::SPW + ln.grp) * C::SV + ln.eq];
      axpy_row<C::NP>(fphi + g * C::NPP, f, acc);
    }
  }
  __syncwarp();
}

// --------------------------------------------------------------- kernels
// One color: surfaces [begin, end) of the color-major list.
template <class C, int PH, bool kRK>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
k_surface_colored(View v, double* __restrict__ U, double* __restrict__ R, RK rk, int64_t begin,
                  int64_t end) {
  extern __shared__ double sm[];
  double* st = sm;
  stage_tables<C>(v.tables, st);
  const Lane ln = lane_info<C>();
  double* ws = sm + C::S_TOTAL + (threadIdx.x >> 5) * C::W_SIZE;
  int* need = reinterpret_cast<int*>(ws + C::W_FLAG) + C::SPW;
  if constexpr (C::DMMA) {  // CM rows beyond N_p stay zero (B padding of the trace)
    for (int i = ln.lane; i < (4 * C::KT - C::NP) * C::LDB; i += 32)
      ws[C::D_CM + C::NP * C::LDB + i] = 0.0;
    __syncwarp();
  }
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t tile = begin + warp * C::SPW; tile < end; tile += nwarp * C::SPW) {
    const int64_t s = tile + ln.grp;
    const SurfCtx c = load_surface<C>(v, ln, s, end, ws);
    const bool first = c.owner && (c.code & (ln.side ? MC_FLAG_R_FIRST : MC_FLAG_L_FIRST));
    const bool last = c.owner && (c.code & (ln.side ? MC_FLAG_R_LAST : MC_FLAG_L_LAST));
    const int64_t off = int64_t(c.has ? c.e : 0) * v.stride + ln.eq * C::NP;
    double u[C::NP], acc[C::NP];
    if (c.has) {
      load_run<C::NP>(U + off, u);
    } else {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) u[j] = 0.0;
    }
    if (c.owner && !first) {
      load_rw<C::NP>(R + off, acc);
    } else {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
    }
    if (__any_sync(kFull, first)) {
      if (ln.active && ln.eq == 0) {
        need[ln.slot] = first;
        if (first) {
          const double* jp = v.jinv + int64_t(c.e) * (C::DIM * C::DIM);
#pragma unroll
          for (int k = 0; k < C::DIM * C::DIM; ++k)
            ws[C::W_JI + ln.slot * C::JIS + k] = __ldg(jp + k);
        }
      }
      __syncwarp();
      if constexpr (C::DMMA)
        volume_dmma<C, PH>(st, ws, need, u, first && ln.active, ln.lane, v.prm, acc);
      else
        volume_tasks<C, PH, C::ES, C::QC>(st, ws + C::W_VS, ws + C::W_VF, ws + C::W_JI, need, u,
                                          ln.slot, ln.eq, first && ln.active, ln.lane, v.prm, acc);
    }
    surface_tasks<C, PH>(st, ws, ln, c, u, v.prm, acc);
    if (c.owner) {
      if (kRK && last) {
        if (rk.save_u0) store_run<C::NP>(static_cast<double*>(rk.U0) + off, u);
        if (rk.a != 0.0) {
          double u0[C::NP];
          load_run<C::NP>(static_cast<const double*>(rk.U0) + off, u0);
#pragma unroll
          for (int j = 0; j < C::NP; ++j) acc[j] = rk.a * u0[j] + rk.b * fma(rk.dt, acc[j], u[j]);
        } else {
#pragma unroll
          for (int j = 0; j < C::NP; ++j) acc[j] = rk.b * fma(rk.dt, acc[j], u[j]);
        }
        store_run<C::NP>(U + off, acc);
        if (v.send_slot) {
          const int sl = __ldg(v.send_slot + c.e);
          if (sl >= 0)
            store_run<C::NP>(static_cast<double*>(v.send_buf) + int64_t(sl) * v.stride + ln.eq * C::NP,
                             acc);
        }
      } else {
        store_run<C::NP>(R + off, acc);
      }
    }
  }
}

// Volume integral for all owned elements (buffered / atomic strategies):
// NEQ lanes per element, same task scheme.
template <class C, int PH>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
k_volume(View v, const double* __restrict__ U, double* __restrict__ R) {
  extern __shared__ double sm[];
  double* st = sm;
  stage_tables<C>(v.tables, st);
  double* ws = sm + C::S_TOTAL + (threadIdx.x >> 5) * C::V_SIZE;
  int* need = reinterpret_cast<int*>(ws + C::V_FLAG);
  const int lane = threadIdx.x & 31;
  int slot = lane / C::NEQ;
  const int eq = lane - slot * C::NEQ;
  const bool act = slot < C::EPW;
  if (!act) slot = 0;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t tile = warp * C::EPW; tile < v.n_elements; tile += nwarp * C::EPW) {
    const int64_t e = tile + slot;
    const bool has = act && e < v.n_elements;
    const int64_t off = (has ? e : 0) * v.stride + eq * C::NP;
    double u[C::NP], acc[C::NP];
    if (has) {
      load_run<C::NP>(U + off, u);
    } else {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) u[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
    if (act && eq == 0) {
      need[slot] = has;
      if (has) {
#pragma unroll
        for (int k = 0; k < C::DIM * C::DIM; ++k)
          ws[C::V_JI + slot * C::JIS + k] = __ldg(v.jinv + e * (C::DIM * C::DIM) + k);
      }
    }
    __syncwarp();
    volume_tasks<C, PH, C::EPW, C::QCV>(st, ws + C::V_VS, ws + C::V_VF, ws + C::V_JI, need, u,
                                        slot, eq, has, lane, v.prm, acc);
    if (has) store_run<C::NP>(R + off, acc);
  }
}

// Surface contributions of ALL surfaces (no coloring) to either the
// 2*ns buffer (kAtomic = false: slot 2s+side) or atomically into R.
template <class C, int PH, bool kAtomic>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
k_surface_uncolored(View v, const double* __restrict__ U, double* __restrict__ out) {
  extern __shared__ double sm[];
  double* st = sm;
  stage_tables<C>(v.tables, st);
  const Lane ln = lane_info<C>();
  double* ws = sm + C::S_TOTAL + (threadIdx.x >> 5) * C::W_SIZE;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t end = v.n_surfaces;
  for (int64_t tile = warp * C::SPW; tile < end; tile += nwarp * C::SPW) {
    const int64_t s = tile + ln.grp;
    const SurfCtx c = load_surface<C>(v, ln, s, end, ws);
    double u[C::NP], acc[C::NP];
    if (c.has) {
      load_run<C::NP>(U + int64_t(c.e) * v.stride + ln.eq * C::NP, u);
    } else {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) u[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
    surface_tasks<C, PH>(st, ws, ln, c, u, v.prm, acc);
    if (kAtomic) {
      if (c.owner) {
        double* dst = out + int64_t(c.e) * v.stride + ln.eq * C::NP;
#pragma unroll
        for (int j = 0; j < C::NP; ++j) atomicAdd(dst + j, acc[j]);
      }
    } else if (c.valid) {
      // buffer slot 2s+side holds this side's contribution (0 if absent)
      double* dst = out + (2 * s + ln.side) * v.stride + ln.eq * C::NP;
      if (!c.owner) {
#pragma unroll
        for (int j = 0; j < C::NP; ++j) acc[j] = 0.0;
      }
      store_run<C::NP>(dst, acc);
    }
  }
}

constexpr int kThreads = 256;

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

}  // namespace mcdg
