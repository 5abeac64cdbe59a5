// Register-resident DG kernels: H lanes per element side (H = 1 or 2).
//
// Lanes (2H*i + H*side + h) serve surface i of a warp (16/H surfaces per
// warp): `side` picks the left / right element, `h` picks an equation group
// (equations [h*NEQH, min(NEQ, (h+1)*NEQH)) ), so a lane holds NEQH*N_p
// coefficients of ONE element in registers:
//   H = 1 when N_eq*N_p <= 24 (c1, c2 Euler p=2 triangles, quad p=1, ...):
//         the whole block, 256-bit loads/stores;
//   H = 2 when N_eq*N_p <= 64 (c3 quad p=3, c4 tet p=2, ...): an equation
//         group, 128-bit loads/stores.
// Per quadrature point a lane evaluates the traces of its own equations,
// assembles the full state of its side from its sibling and the other
// side's state from the partner lane (warp shuffles), evaluates the
// Lax-Friedrichs flux (all 2H lanes of a surface compute the same value —
// redundant but register-only), and lifts its own equations into its
// residual block.  In the first-touch pass it also evaluates the element's
// volume integral the same way.  Reference-element tables live in shared
// memory (volume tables are warp-wide broadcasts, face tables are indexed by
// the side code); no per-element data ever goes through shared memory,
// which is what keeps these kernels off the shared-memory roofline that
// bounds the group kernel (dg_kernels.cuh).
//
// Same accumulation order per element as Algorithm 1 and the oracle:
// volume, then colors 1..n; within a surface the quadrature points in order.
#pragma once

#include "dg_kernels.cuh"

namespace mcdg {

template <class C>
struct Tpe {
  static constexpr int W = C::NEQ * C::NP;
  static constexpr int H = (W <= 24) ? 1 : ((W <= 64 && C::NEQ >= 2) ? 2 : 0);
  static constexpr int NEQH = H ? (C::NEQ + H - 1) / H : C::NEQ;   // eqs of lane h = 0
  static constexpr int NEQ1 = C::NEQ - NEQH;
  // H = 2: lane h = 0 holds equations [0, NA), lane h = 1 holds [NA, NEQ)
  // (NA <= NEQH: with an odd count the second lane takes the larger group,
  // so both runs start 32-byte aligned for tets, 2 + 3 equations x 10)
  static constexpr int NA = (H == 2) ? NEQ1 : NEQH;
  static constexpr int WH = NEQH * C::NP;                          // doubles per lane
  // H = 2 moves 16-byte pairs: every lane's run must have even length
  static constexpr bool PAIRS = (C::NP % 2 == 0) || (NEQH % 2 == 0 && NEQ1 % 2 == 0);
#ifdef MC_TPE_H1_ONLY
  static constexpr bool OK = H == 1;
#else
#ifdef MC_TET_GROUP
  static constexpr bool OK = H == 1 || (H == 2 && PAIRS && C::DIM == 2);
#else
  // tets too since the volume tables moved to constant memory (c4: 1.01 vs
  // 0.93 G edges/s for the group kernel); MC_TET_GROUP restores the latter
  static constexpr bool OK = H == 1 || (H == 2 && PAIRS);
#endif
#endif
  // 256-bit accesses for every lane's run: 32-byte aligned offsets and
  // lengths (blocks are 32-byte padded); H = 2 when both equation groups
  // span a multiple of four coefficients (c3: 2 x 16)
  static constexpr bool V4 = (H == 1 && W % 4 == 0) ||
                             (H == 2 && (NA * C::NP) % 4 == 0 && (NEQH * C::NP) % 2 == 0);
  static constexpr int SW = 16 / (H ? H : 1);                      // surfaces per warp
  static constexpr int THREADS = 128;
#ifdef MC_MINB_TPE
  static constexpr int MINB = MC_MINB_TPE;
#else
  static constexpr int MINB = (H == 2) ? 2 : ((W > 16) ? 3 : 4);
#endif
  // two lanes per side on tets: fluxes as warp tasks (c4 1.17 -> 1.22 G
  // edges/s); quads keep the per-lane flux (c3 neutral, its first-touch
  // color slower).  MC_NO_H2_TASKS / MC_H2_TASKS_ALL for A/B.
#if defined(MC_NO_H2_TASKS)
  static constexpr bool TASKS = false;
#elif defined(MC_H2_TASKS_ALL)
  static constexpr bool TASKS = (H == 2);
#else
  static constexpr bool TASKS = (H == 2 && C::DIM == 3);
#endif
  // per-warp scratch of the task-packed surface flux (TASKS): traces
  // [NQF][SW][2][SV], canonical fluxes [NQF][SW][SV], normals [SW][DIM],
  // flags [SW] (ints); SV odd
  static constexpr int SV = C::NEQ | 1;
  static constexpr int X_TR = 0;
  static constexpr int X_FS = X_TR + C::NQF * (16 / (H ? H : 1)) * 2 * SV;
  static constexpr int X_NRM = X_FS + C::NQF * (16 / (H ? H : 1)) * SV;
  static constexpr int X_FLG = X_NRM + (16 / (H ? H : 1)) * C::DIM;
  static constexpr int X_SIZE = (X_FLG + (16 / (H ? H : 1)) / 2 + 2) & ~1;
  // two-lane 2D kernels: task-packed fluxes in the surface-only and
  // last-touch passes only (c3 surface colors +2.5 %); their first-touch
  // pass keeps the per-lane flux and the small shared-memory footprint.
  // MC_NO_SURF_TASKS for A/B.
#ifdef MC_NO_SURF_TASKS
  static constexpr bool TASKS_SURF = TASKS;
#else
  // only when the (surface, point) tasks fill the warp: 3-point edges (p =
  // 2 quads, hybrid meshes) leave a quarter of the lanes idle and measured
  // slower (h1 1.29 -> 1.35 G edges/s with per-lane fluxes)
  static constexpr bool TASKS_SURF = TASKS || (H == 2 && (16 / (H ? H : 1)) * C::NQF >= 32);
#endif
  static constexpr int SMEM = (C::S_TOTAL + (TASKS ? 4 * X_SIZE : 0)) * 8;
  static constexpr int SMEM_SURF = (C::S_TOTAL + (TASKS_SURF ? 4 * X_SIZE : 0)) * 8;
};

template <int NP, int N>
__device__ __forceinline__ double tdot(const double* row, const double (&u)[N], int off) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < NP / 2; ++j) {
    const double2 a = r2[j];
    t = fma(a.x, u[off + 2 * j], t);
    t = fma(a.y, u[off + 2 * j + 1], t);
  }
  if constexpr (NP % 2) t = fma(row[NP - 1], u[off + NP - 1], t);
  return t;
}

// As tdot with two partial sums (even / odd j): half the dependent-FMA
// chain, for latency-bound trace loops
template <int NP, int N>
__device__ __forceinline__ double tdot2(const double* row, const double (&u)[N], int off) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  double t0 = 0.0, t1 = 0.0;
#pragma unroll
  for (int j = 0; j < NP / 2; ++j) {
    const double2 a = r2[j];
    t0 = fma(a.x, u[off + 2 * j], t0);
    t1 = fma(a.y, u[off + 2 * j + 1], t1);
  }
  if constexpr (NP % 2) t0 = fma(row[NP - 1], u[off + NP - 1], t0);
  return t0 + t1;
}

template <int NP, int N>
__device__ __forceinline__ void taxpy(const double* row, double f, double (&acc)[N], int off) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int j = 0; j < NP / 2; ++j) {
    const double2 a = r2[j];
    acc[off + 2 * j] = fma(a.x, f, acc[off + 2 * j]);
    acc[off + 2 * j + 1] = fma(a.y, f, acc[off + 2 * j + 1]);
  }
  if constexpr (NP % 2) acc[off + NP - 1] = fma(row[NP - 1], f, acc[off + NP - 1]);
}

// Full state of this side at one point from the lanes' own traces.
template <class C>
__device__ __forceinline__ void assemble_state(const double (&own)[Tpe<C>::NEQH], int h,
                                               double (&s)[C::NEQ]) {
  constexpr int NEQH = Tpe<C>::NEQH;
  if constexpr (Tpe<C>::H == 1) {
#pragma unroll
    for (int k = 0; k < C::NEQ; ++k) s[k] = own[k];
  } else {
    double oth[NEQH];
#pragma unroll
    for (int k = 0; k < NEQH; ++k) oth[k] = __shfl_xor_sync(kFull, own[k], 1);
    constexpr int NA = Tpe<C>::NA;
#pragma unroll
    for (int e = 0; e < C::NEQ; ++e)
      s[e] = (e < NA) ? (h == 0 ? own[e] : oth[e])
                      : (h == 1 ? own[e - NA] : oth[e - NA]);
  }
}

// This lane's k-th equation of a full NEQ vector.
template <class C>
__device__ __forceinline__ double own_part(const double* v, int h, int k) {
  constexpr int NEQH = Tpe<C>::NEQH;
  if constexpr (Tpe<C>::H == 1) {
    return v[k];
  } else {
    constexpr int NA = Tpe<C>::NA;
    const int e1 = (NA + k < C::NEQ) ? NA + k : C::NEQ - 1;
    return h == 0 ? v[k] : v[e1];
  }
}

// volume-point loop unroll: 2 for two lanes per side (c3 1.12 -> 1.15 G
// edges/s, c4 neutral), 1 for one lane (registers); MC_VOL_UNROLL overrides
#ifdef MC_VOL_UNROLL
template <int H> constexpr int kVolUnroll = MC_VOL_UNROLL;
#else
template <int H> constexpr int kVolUnroll = H == 2 ? 2 : 1;
#endif

#ifdef MC_P1PROJ_H1
constexpr bool kP1ProjH1 = true;
#else
constexpr bool kP1ProjH1 = false;
#endif

// Balanced volume lanes (MC_VOL_BAL; two lanes per side, odd N_eq: lane 0
// holds NA equations, lane 1 NA + 1): for the volume integral lane 0 also
// loads the last equation into its spare slot NA, and at each point pair
// each lane evaluates that equation's trace and projection at its OWN point
// only (the two partial moments are summed once at the end): 5 instead of
// 6 trace and projection runs per lane and pair on c4.
template <class C>
constexpr bool kVolBal =
#ifndef MC_VOL_BAL
    false &&
#endif
    Tpe<C>::H == 2 && C::P1PROJ && Tpe<C>::NEQH == Tpe<C>::NA + 1;

// Mode-split projection (two lanes per side, even NPL): at each point pair
// both lanes hold the full flux of their own point; lane h accumulates the
// P_{p-1} modes [h*NPL/2, (h+1)*NPL/2) of ALL equations at both points (the
// partner's fluxes cross by one shuffle each), so the projection needs no
// per-component selects and no dead spare-slot equation; the two mode halves
// of each lane's own equations cross once per element before the lift.
template <class C>
constexpr bool kVolMsplit =
#ifdef MC_VOL_NO_MSPLIT
    false &&
#endif
    Tpe<C>::H == 2 && C::P1PROJ && C::NPL % 2 == 0;

// Modes of P_d on the simplex (d < 0: none) and the P_{p-1} modes the
// reference gradient of mode j needs (modes are ordered by total degree).
template <int K>
constexpr int simplex_modes(int d) {
  return d < 0 ? 0 : (K == TRI ? (d + 1) * (d + 2) / 2 : (d + 1) * (d + 2) * (d + 3) / 6);
}
template <int K>
constexpr int grad_shell(int j) {
  int d = 0;
  while (j >= simplex_modes<K>(d)) ++d;
  return simplex_modes<K>(d - 1);
}

// Volume integral through P_{p-1} (Cfg::P1PROJ, simplices): the physical
// fluxes are first projected onto the NPL modes of P_{p-1} with the weights
// folded in (Pd[d][k][m] = sum_q w_q phi_m(q) F_d(q)[k]), the element's
// (constant) inverse Jacobian turns them into contravariant moments once,
// Pm[r] = sum_d Jinv[r][d] Pd[d], and they are lifted once per element,
// acc[k][j] += sum_r sum_m D_r[j][m] Pm[r][k][m], with D's zero blocks
// skipped at compile time (c4: 3 x 4 instead of 3 x 10 multiply-adds per
// point and equation, no Jacobian per point).  Two lanes per side also
// split the volume points: at each point pair, lane h evaluates the flux
// of point 2i+h only (the traces and the fluxes of the other lane's
// equations cross by shuffles), so every flux is evaluated once, not twice.
template <class C, int PH>
__device__ __forceinline__ void tpe_volume_p1(const double* vphi, const double* svphi,
                                              const double (&u)[Tpe<C>::WH],
                                              const double* __restrict__ jinv_e, int h,
                                              int nown, bool mine, const Params& P,
                                              double (&acc)[Tpe<C>::WH],
                                              double* jst = nullptr) {
  constexpr int NP = C::NP, NEQ = C::NEQ, NEQH = Tpe<C>::NEQH, DIM = C::DIM, M = C::NPL;
  constexpr int H = Tpe<C>::H, WH = Tpe<C>::WH;
  const double* wpsi = vphi + (C::S_WPSI - C::S_VPHI);
  const double* dmat = vphi + (C::S_DMAT - C::S_VPHI);
  // the Jacobian is needed only at the end: either copied asynchronously
  // into the warp scratch now (jst: this side's DIM^2 slot, the side's H
  // lanes split the copies; cp.async, no registers held) or its line
  // pulled into L1
  if (jst) {
    constexpr int JN = DIM * DIM, PER = (JN + H - 1) / H;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int k = h * PER + i;
      if (k < JN) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(jst + k));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(jinv_e + k)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(jinv_e));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(jinv_e + DIM * DIM - 1));
  }
  double Pm[DIM][NEQH][M];
#pragma unroll
  for (int r = 0; r < DIM; ++r)
#pragma unroll
    for (int k = 0; k < NEQH; ++k)
#pragma unroll
      for (int m = 0; m < M; ++m) Pm[r][k][m] = 0.0;
  // whole point on this lane: every own equation's flux at point q
  auto point = [&](int q) {
    double own[NEQH], s[NEQ];
#pragma unroll
    for (int k = 0; k < NEQH; ++k) own[k] = tdot<NP, WH>(vphi + q * C::NPP, u, k * NP);
    assemble_state<C>(own, h, s);
    double F[DIM * NEQ];
    Physics<PH, DIM, NEQ>::pflux(s, P, F);
#pragma unroll
    for (int d = 0; d < DIM; ++d)
#pragma unroll
      for (int k = 0; k < NEQH; ++k) {
        const double f = (mine && k < nown) ? own_part<C>(F + d * NEQ, h, k) : 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) Pm[d][k][m] = fma(wpsi[q * M + m], f, Pm[d][k][m]);
      }
  };
  auto load_ji = [&](double (&ji)[DIM * DIM]) {
    if (jst) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int k = 0; k < DIM * DIM; ++k) ji[k] = jst[k];
    } else {
#pragma unroll
      for (int k = 0; k < DIM * DIM; ++k) ji[k] = __ldg(jinv_e + k);
    }
  };
  if constexpr (H == 1) {
#pragma unroll 1
    for (int q = 0; q < C::NQV; ++q) point(q);
  } else if constexpr (kVolMsplit<C>) {
    constexpr int NA = Tpe<C>::NA, MH = M / 2;
    // this lane's modes of the weighted P_{p-1} table (shared-memory copy:
    // the row depends on the lane)
    const double* wmine = svphi + (C::S_WPSI - C::S_VPHI) + h * MH;
    double Q[DIM][NEQ][MH];
#pragma unroll
    for (int d = 0; d < DIM; ++d)
#pragma unroll
      for (int k = 0; k < NEQ; ++k)
#pragma unroll
        for (int m = 0; m < MH; ++m) Q[d][k][m] = 0.0;
#ifndef MC_MSPLIT_UNROLL
#define MC_MSPLIT_UNROLL 1
#endif
    constexpr int kMsUnroll = MC_MSPLIT_UNROLL;
#pragma unroll kMsUnroll
    for (int q0 = 0; q0 + 1 < C::NQV; q0 += 2) {
      const int q1 = q0 + 1;
      const int qm = q0 + h, qo = q1 - h;
      // balanced lanes (kVolBal): the shared equations at both points, the
      // last one (both lanes hold it in slot NA) at this lane's point only
      constexpr int NT = kVolBal<C> ? NA : NEQH;
      double mt[NEQH], ot[NEQH];
#ifdef MC_VOL_TRACE_SMEM   // lane-dependent rows from the shared copy: no selects
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        ot[k] = __shfl_xor_sync(kFull, tdot<NP, WH>(svphi + qo * C::NPP, u, k * NP), 1);
        mt[k] = tdot<NP, WH>(svphi + qm * C::NPP, u, k * NP);
      }
#else
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double a = tdot<NP, WH>(vphi + q0 * C::NPP, u, k * NP);
        const double b = tdot<NP, WH>(vphi + q1 * C::NPP, u, k * NP);
        ot[k] = __shfl_xor_sync(kFull, h ? a : b, 1);
        mt[k] = h ? b : a;
      }
#endif
      double s[NEQ], F[DIM * NEQ];
#pragma unroll
      for (int e = 0; e < NEQ; ++e)
        s[e] = (e < NA) ? (h == 0 ? mt[e] : ot[e]) : (h == 1 ? mt[e - NA] : ot[e - NA]);
      if constexpr (kVolBal<C>) s[NEQ - 1] = tdot<NP, WH>(svphi + qm * C::NPP, u, NA * NP);
      Physics<PH, DIM, NEQ>::pflux(s, P, F);
      double wm[MH], wo[MH];
#pragma unroll
      for (int m = 0; m < MH; ++m) {
        wm[m] = wmine[qm * M + m];
        wo[m] = wmine[qo * M + m];
      }
      // idle lane pairs accumulate garbage that never leaves the pair (as
      // in the equation-split loop below)
#pragma unroll
      for (int d = 0; d < DIM; ++d)
#pragma unroll
        for (int k = 0; k < NEQ; ++k) {
          const double fm = F[d * NEQ + k];
          const double fo = __shfl_xor_sync(kFull, fm, 1);
#pragma unroll
          for (int m = 0; m < MH; ++m) Q[d][k][m] = fma(wo[m], fo, fma(wm[m], fm, Q[d][k][m]));
        }
    }
    if constexpr (C::NQV % 2) {   // last point: both lanes evaluate it
      constexpr int q = C::NQV - 1;
      double own[NEQH], s[NEQ], F[DIM * NEQ];
#pragma unroll
      for (int k = 0; k < NEQH; ++k) own[k] = tdot<NP, WH>(vphi + q * C::NPP, u, k * NP);
      assemble_state<C>(own, h, s);
      Physics<PH, DIM, NEQ>::pflux(s, P, F);
#pragma unroll
      for (int d = 0; d < DIM; ++d)
#pragma unroll
        for (int k = 0; k < NEQ; ++k)
#pragma unroll
          for (int m = 0; m < MH; ++m) Q[d][k][m] = fma(wmine[q * M + m], F[d * NEQ + k], Q[d][k][m]);
    }
    double ji[DIM * DIM];
    load_ji(ji);
#pragma unroll
    for (int k = 0; k < NEQ; ++k)
#pragma unroll
      for (int m = 0; m < MH; ++m) {
        double pd[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) pd[d] = Q[d][k][m];
#pragma unroll
        for (int r = 0; r < DIM; ++r) {
          double t = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) t = fma(ji[r * DIM + d], pd[d], t);
          Q[r][k][m] = t;
        }
      }
    // my equations' contravariant moments: my mode half, the partner's by
    // shuffle (lane 0 holds modes [0, MH), lane 1 [MH, M))
#pragma unroll
    for (int r = 0; r < DIM; ++r)
#pragma unroll
      for (int k = 0; k < NEQH; ++k) {
        const int k1 = (NA + k < NEQ) ? NA + k : NEQ - 1;   // lane 1's slot-k equation
#pragma unroll
        for (int m = 0; m < MH; ++m) {
          const double q0v = Q[r][k][m], q1v = Q[r][k1][m];
          const double mine_v = h ? q1v : q0v;
          const double recv = __shfl_xor_sync(kFull, h ? q0v : q1v, 1);
          Pm[r][k][m] = h ? recv : mine_v;
          Pm[r][k][MH + m] = h ? mine_v : recv;
        }
      }
  } else if constexpr (kVolBal<C>) {
    // slot NA holds the last equation on both lanes; its table rows and
    // weights are lane-dependent (my point), read from the shared-memory
    // copy (rows 2i and 2i+1 sit in different banks)
    constexpr int NA = Tpe<C>::NA;
    const double* swpsi = svphi + (C::S_WPSI - C::S_VPHI);
    static_assert(C::NQV % 2 == 0, "balanced volume lanes take point pairs");
#pragma unroll 1
    for (int q0 = 0; q0 < C::NQV; q0 += 2) {
      const int q1 = q0 + 1, qm = q0 + h;
      double mt[NA], ot[NA];
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        const double a = tdot<NP, WH>(vphi + q0 * C::NPP, u, k * NP);
        const double b = tdot<NP, WH>(vphi + q1 * C::NPP, u, k * NP);
        ot[k] = __shfl_xor_sync(kFull, h ? a : b, 1);
        mt[k] = h ? b : a;
      }
      const double last = tdot<NP, WH>(svphi + qm * C::NPP, u, NA * NP);
      double s[NEQ], F[DIM * NEQ];
#pragma unroll
      for (int e = 0; e < NEQ - 1; ++e)
        s[e] = (e < NA) ? (h == 0 ? mt[e] : ot[e]) : (h == 1 ? mt[e - NA] : ot[e - NA]);
      s[NEQ - 1] = last;
      Physics<PH, DIM, NEQ>::pflux(s, P, F);
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          const double fm = h ? F[d * NEQ + NA + k] : F[d * NEQ + k];
          const double fr = __shfl_xor_sync(kFull, h ? F[d * NEQ + k] : F[d * NEQ + NA + k], 1);
          const double f0 = mine ? (h ? fr : fm) : 0.0;
          const double f1 = mine ? (h ? fm : fr) : 0.0;
#pragma unroll
          for (int m = 0; m < M; ++m)
            Pm[d][k][m] = fma(wpsi[q1 * M + m], f1, fma(wpsi[q0 * M + m], f0, Pm[d][k][m]));
        }
        const double fl = mine ? F[d * NEQ + NEQ - 1] : 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) Pm[d][NA][m] = fma(swpsi[qm * M + m], fl, Pm[d][NA][m]);
      }
    }
#pragma unroll
    for (int d = 0; d < DIM; ++d)
#pragma unroll
      for (int m = 0; m < M; ++m)
        Pm[d][NA][m] += __shfl_xor_sync(kFull, Pm[d][NA][m], 1);
  } else {
    constexpr int NA = Tpe<C>::NA;
#ifndef MC_PAIR_UNROLL
#define MC_PAIR_UNROLL 1
#endif
    constexpr int kPairUnroll = MC_PAIR_UNROLL;
#pragma unroll kPairUnroll
    for (int q0 = 0; q0 + 1 < C::NQV; q0 += 2) {
      const int q1 = q0 + 1;
      double mt[NEQH], ot[NEQH];
#pragma unroll
      for (int k = 0; k < NEQH; ++k) {
        const double a = tdot<NP, WH>(vphi + q0 * C::NPP, u, k * NP);
        const double b = tdot<NP, WH>(vphi + q1 * C::NPP, u, k * NP);
        ot[k] = __shfl_xor_sync(kFull, h ? a : b, 1);    // partner's traces at my point
        mt[k] = h ? b : a;                                // mine at my point (q0 + h)
      }
      double s[NEQ], F[DIM * NEQ];
#pragma unroll
      for (int e = 0; e < NEQ; ++e)
        s[e] = (e < NA) ? (h == 0 ? mt[e] : ot[e]) : (h == 1 ? mt[e - NA] : ot[e - NA]);
      Physics<PH, DIM, NEQ>::pflux(s, P, F);
      // weights of my point and of the partner's (selected once per pair,
      // not per flux component).  Lanes whose element takes no volume
      // term here (not first touch, no element) accumulate garbage that
      // never leaves the lane pair and is never stored: the caller
      // replaces their acc (residual load) or does not store it.
#ifdef MC_PAIR_WSEL   // weights selected once per pair: more registers, c4 -10 %
      double wm[M], wo[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const double w0 = wpsi[q0 * M + m], w1 = wpsi[q1 * M + m];
        wm[m] = h ? w1 : w0;
        wo[m] = h ? w0 : w1;
      }
#pragma unroll
      for (int d = 0; d < DIM; ++d)
#pragma unroll
        for (int k = 0; k < NEQH; ++k) {
          const double fm = own_part<C>(F + d * NEQ, h, k);         // my eq, my point
          const double fr = __shfl_xor_sync(kFull, own_part<C>(F + d * NEQ, h ^ 1, k), 1);
#pragma unroll
          for (int m = 0; m < M; ++m) Pm[d][k][m] = fma(wo[m], fr, fma(wm[m], fm, Pm[d][k][m]));
        }
#else   // per-component selects of the two points' fluxes (measured faster)
#pragma unroll
      for (int d = 0; d < DIM; ++d)
#pragma unroll
        for (int k = 0; k < NEQH; ++k) {
          const double fm = own_part<C>(F + d * NEQ, h, k);
          const double fr = __shfl_xor_sync(kFull, own_part<C>(F + d * NEQ, h ^ 1, k), 1);
#ifndef MC_PAIR_ZERO_IDLE   // no zeroing (c4 color 1 +1.6 %): garbage stays in
                            // non-contributing lane pairs, whose acc is replaced
                            // (residual load) or never stored
          const double f0 = h ? fr : fm;
          const double f1 = h ? fm : fr;
#else
          const bool on = mine && k < nown;
          const double f0 = on ? (h ? fr : fm) : 0.0;
          const double f1 = on ? (h ? fm : fr) : 0.0;
#endif
#pragma unroll
          for (int m = 0; m < M; ++m)
            Pm[d][k][m] = fma(wpsi[q1 * M + m], f1, fma(wpsi[q0 * M + m], f0, Pm[d][k][m]));
        }
#endif
    }
    if constexpr (C::NQV % 2) point(C::NQV - 1);
  }
  // physical -> contravariant moments with the element's inverse Jacobian
  // (the mode-split branch has done it on its own layout)
  if constexpr (!kVolMsplit<C>) {
  double ji[DIM * DIM];
  load_ji(ji);
#pragma unroll
  for (int k = 0; k < NEQH; ++k)
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double pd[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) pd[d] = Pm[d][k][m];
#pragma unroll
      for (int r = 0; r < DIM; ++r) {
        double t = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) t = fma(ji[r * DIM + d], pd[d], t);
        Pm[r][k][m] = t;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NEQH; ++k)
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      double a = acc[k * NP + j];
#pragma unroll
      for (int r = 0; r < DIM; ++r)
#pragma unroll
        for (int m = 0; m < grad_shell<C::KIND>(j); ++m)
          a = fma(dmat[(r * NP + j) * M + m], Pm[r][k][m], a);
      acc[k * NP + j] = a;
    }
}

// Volume integral of this lane's element (its equations), added into acc.
template <class C, int PH>
__device__ __forceinline__ void tpe_volume(const double* st, const double (&u)[Tpe<C>::WH],
                                           const double* __restrict__ jinv_e, int h, int nown,
                                           bool mine, const Params& P,
                                           double (&acc)[Tpe<C>::WH], int ek = 0,
                                           double* jst = nullptr) {
  constexpr int WH = Tpe<C>::WH, NP = C::NP, NEQ = C::NEQ, NEQH = Tpe<C>::NEQH, DIM = C::DIM;
  const double* vphi = vol_tables<C, true>(st);
  const double* vdphi = vphi + (C::S_VDPHI - C::S_VPHI);
  const double* vw = vphi + (C::S_VW - C::S_VPHI);
  // two lanes per side (tets): c4 first-touch color 4.91 -> 4.57 ms; one
  // lane (c2 triangles) measured slower (color 1 3.55 -> 3.27 TB/s)
  if constexpr (C::P1PROJ && (Tpe<C>::H == 2 || kP1ProjH1)) {
    tpe_volume_p1<C, PH>(vphi, st + C::S_VPHI, u, jinv_e, h, nown, mine, P, acc, jst);
    return;
  }
  double ji[DIM * DIM];
#pragma unroll
  for (int k = 0; k < DIM * DIM; ++k) ji[k] = __ldg(jinv_e + k);
  // tensor-product quads (QUAD, and the quads of a HYB mesh): sum
  // factorisation (basis l_i(x) l_j(y), Gauss points (x_a, y_b)), half the
  // multiply-adds of the dense contraction.
  //   trace:      T[j] = sum_i l_i(x_a) u[i][j];  U(a,b) = sum_j l_j(y_b) T[j]
  //   projection: A[j] += w_ab l_j(y_b) F0, B[j] += w_ab l'_j(y_b) F1 over b,
  //               then acc[i][j] += l'_i(x_a) A[j] + l_i(x_a) B[j]
  // The 1D values are entries of the 2D tables (l_0 = 1 for the
  // orthonormal basis on [0,1]); `onk` = this lane's element is a quad.
  auto quad_sf = [&](bool onk) {
    if constexpr (C::KIND == QUAD || C::KIND == HYB) {
    constexpr int n = C::PDEG + 1;
    static_assert(n * n == NP && n * n == C::NQV_QUAD, "tensor quad layout");
    auto L1 = [&](int a, int i) { return vphi[(a * n) * C::NPP + i * n]; };
    auto D1 = [&](int a, int i) { return vdphi[(a * n) * C::NPP + i * n]; };
#pragma unroll 1
    for (int a = 0; a < n; ++a) {
      double T[NEQH][n], A[NEQH][n], B[NEQH][n];
#pragma unroll
      for (int k = 0; k < NEQH; ++k)
#pragma unroll
        for (int j = 0; j < n; ++j) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) t = fma(L1(a, i), u[k * NP + i * n + j], t);
          T[k][j] = t;
          A[k][j] = 0.0;
          B[k][j] = 0.0;
        }
#pragma unroll
      for (int b = 0; b < n; ++b) {
        double own[NEQH], s[NEQ], Ft[DIM * NEQ];
#pragma unroll
        for (int k = 0; k < NEQH; ++k) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < n; ++j) t = fma(L1(b, j), T[k][j], t);
          own[k] = t;
        }
        assemble_state<C>(own, h, s);
        Physics<PH, DIM, NEQ>::vflux(s, ji, P, Ft);
        const double w = vw[a * n + b];
#pragma unroll
        for (int k = 0; k < NEQH; ++k) {
          const bool on = mine && onk && k < nown;
          const double g0 = on ? w * own_part<C>(Ft, h, k) : 0.0;
          const double g1 = on ? w * own_part<C>(Ft + NEQ, h, k) : 0.0;
#pragma unroll
          for (int j = 0; j < n; ++j) {
            A[k][j] = fma(L1(b, j), g0, A[k][j]);
            B[k][j] = fma(D1(b, j), g1, B[k][j]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NEQH; ++k)
#pragma unroll
        for (int i = 0; i < n; ++i)
#pragma unroll
          for (int j = 0; j < n; ++j)
            acc[k * NP + i * n + j] =
                fma(D1(a, i), A[k][j], fma(L1(a, i), B[k][j], acc[k * NP + i * n + j]));
    }
    }
  };
#ifndef MC_NO_QUAD_SF
  if constexpr (C::KIND == QUAD && Tpe<C>::H == 2) {
    quad_sf(true);
    return;
  }
#endif
  constexpr int kUnroll = kVolUnroll<Tpe<C>::H>;
  // volume points [qa, qb) of the tables; `on` = this lane's element uses
  // them (HYB: the quad rule's rows, then the triangle rule's)
  auto points = [&](int qa, int qb, bool on) {
#pragma unroll kUnroll
  for (int q = qa; q < qb; ++q) {
    double own[NEQH], s[NEQ];
#pragma unroll
    for (int k = 0; k < NEQH; ++k) own[k] = tdot<NP, WH>(vphi + q * C::NPP, u, k * NP);
    assemble_state<C>(own, h, s);
    const double w = vw[q];
    if constexpr (Tpe<C>::H == 1 && PH == EULER) {
      // whole block in this lane: fluxes straight into the projection
      const double inv = flux_rcp<true>(s[0]);
      double vel[DIM], ke = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        vel[d] = s[1 + d] * inv;
        ke += s[1 + d] * vel[d];
      }
      const double p = (P.gamma - 1.0) * (s[NEQ - 1] - 0.5 * ke);
#pragma unroll
      for (int r = 0; r < DIM; ++r) {
        double ut = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) ut += ji[r * DIM + d] * vel[d];
        const double* dp = vdphi + (r * C::NQV + q) * C::NPP;
        taxpy<NP, WH>(dp, w * (s[0] * ut), acc, 0);
#pragma unroll
        for (int d = 0; d < DIM; ++d)
          taxpy<NP, WH>(dp, w * (s[1 + d] * ut + p * ji[r * DIM + d]), acc, (1 + d) * NP);
        taxpy<NP, WH>(dp, w * ((s[NEQ - 1] + p) * ut), acc, (NEQ - 1) * NP);
      }
    } else {
      double Ft[DIM * NEQ];
      Physics<PH, DIM, NEQ>::vflux(s, ji, P, Ft);
#pragma unroll
      for (int r = 0; r < DIM; ++r) {
        const double* dp = vdphi + (r * C::NQV + q) * C::NPP;
#pragma unroll
        for (int k = 0; k < NEQH; ++k) {
          // uniform control flow (zero factor for idle lanes) keeps the
          // constant-memory table reads warp-uniform (c3: 0.94 -> 0.97)
          const double f = (mine && on && k < nown) ? w * own_part<C>(Ft + r * NEQ, h, k) : 0.0;
          taxpy<NP, WH>(dp, f, acc, k * NP);
        }
      }
    }
  }
  };
  if constexpr (C::KIND == HYB) {
    // conforming triangle + quad mix: each element integrates with its own
    // kind's rule and basis (triangle rows are zero beyond its N_p)
    if constexpr (Tpe<C>::H == 1) {   // called per lane (no shuffles)
      if (ek) points(0, C::NQV_QUAD, true);
      else points(C::NQV_QUAD, C::NQV, true);
    } else {                          // the whole warp takes part (shuffles)
      if (__any_sync(kFull, mine && ek)) {
#ifndef MC_NO_QUAD_SF
        quad_sf(ek != 0);
#else
        points(0, C::NQV_QUAD, ek != 0);
#endif
      }
      if (__any_sync(kFull, mine && !ek)) points(C::NQV_QUAD, C::NQV, ek == 0);
    }
  } else {
    points(0, C::NQV, true);
  }
}


// lane 0's spare equation slot NA of its coefficient array (kVolBal)
template <class C>
__device__ __forceinline__ double (&bal_slot(double (&u)[Tpe<C>::WH]))[C::NP] {
  return *reinterpret_cast<double(*)[C::NP]>(&u[Tpe<C>::NA * C::NP]);
}

struct TpeSide {
  int e, mycode;
  uint32_t code;
  double scale, n[3];
  bool valid, has, owner, boundary;
};

template <class C>
__device__ __forceinline__ TpeSide tpe_side(const View& v, int64_t s, int64_t end, int side) {
  TpeSide t;
  t.valid = s < end;
  int L = 0, R = -1;
  t.code = 0;
  t.scale = 0.0;
  t.n[0] = 1.0;
  t.n[1] = 0.0;
  t.n[2] = 0.0;
  if (t.valid) {
    L = __ldg(v.left + s);
    R = __ldg(v.right + s);
    t.code = __ldg(v.code + s);
    const double* gm = v.geom + s * C::GEOM;
#pragma unroll
    for (int d = 0; d < C::DIM; ++d) t.n[d] = __ldg(gm + d);
    t.scale = __ldg(gm + C::DIM + side);
  }
  t.boundary = R < 0;
  if (v.ghost_par >= 0 && R >= v.n_elements) R = int(v.n_elements + 2 * (R - v.n_elements) + v.ghost_par);
  t.e = side ? R : L;
  t.has = t.valid && t.e >= 0;
  t.owner = t.has && !(side && (t.code & MC_FLAG_R_GHOST));
  t.mycode = side ? int((t.code >> 6) & 63u) : int(t.code & 63u);
  return t;
}

// As tpe_side, with this lane's element id already loaded (one tile ahead:
// the element-block loads of a tile then wait on one DRAM round trip, not
// on the index load and then the block load).
template <class C>
__device__ __forceinline__ TpeSide tpe_side_pre(const View& v, int64_t s, int64_t end, int side,
                                                int e_pre, const uint32_t* code_pre = nullptr) {
  TpeSide t;
  t.valid = s < end;
  t.code = 0;
  t.scale = 0.0;
  t.n[0] = 1.0;
  t.n[1] = 0.0;
  t.n[2] = 0.0;
  if (t.valid) {
    t.code = code_pre ? *code_pre : __ldg(v.code + s);
    const double* gm = v.geom + s * C::GEOM;
#pragma unroll
    for (int d = 0; d < C::DIM; ++d) t.n[d] = __ldg(gm + d);
    t.scale = __ldg(gm + C::DIM + side);
  }
  if (v.ghost_par >= 0 && e_pre >= v.n_elements)   // double-buffered ghost rows
    e_pre = int(v.n_elements + 2 * (e_pre - v.n_elements) + v.ghost_par);
  t.e = t.valid ? e_pre : -1;
  t.boundary = side && t.e < 0;
  t.has = t.valid && t.e >= 0;
  t.owner = t.has && !(side && (t.code & MC_FLAG_R_GHOST));
  t.mycode = side ? int((t.code >> 6) & 63u) : int(t.code & 63u);
  return t;
}

// Lax-Friedrichs flux out of this lane's element with the per-state work
// shared across the surface: each side forms the primitive quantities of
// its OWN state (velocity, pressure, normal velocity, sound speed) and
// takes the other side's (p, c, -v.n) from the partner lane (xor H).  The
// values are bit-identical to evaluating both states here (the partner's
// normal velocity is computed with the negated normal: an exact negation),
// so each lane's result still depends only on its element's view.
template <int PH, int DIM, int NEQ, int H>
__device__ __forceinline__ void lf_shared(const double* s, const double* x, const double* n,
                                          const Params& P, double* out) {
  if constexpr (PH != EULER) {
    Physics<PH, DIM, NEQ>::lf(s, x, n, P, out);
  } else {
    double uo[DIM], po, io;
    Physics<PH, DIM, NEQ>::template prim<true>(s, P, uo, po, io);
    double vo = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) vo += uo[d] * n[d];
    const double co = flux_sqrt<true>(P.gamma * po * io);
    const double vx = -__shfl_xor_sync(kFull, vo, H);
    const double px = __shfl_xor_sync(kFull, po, H);
    const double cx = __shfl_xor_sync(kFull, co, H);
    const double lam = fmax(fabs(vo) + co, fabs(vx) + cx);
    out[0] = 0.5 * (s[0] * vo + x[0] * vx) - 0.5 * lam * (x[0] - s[0]);
#pragma unroll
    for (int d = 0; d < DIM; ++d)
      out[1 + d] = 0.5 * ((s[1 + d] * vo + po * n[d]) + (x[1 + d] * vx + px * n[d])) -
                   0.5 * lam * (x[1 + d] - s[1 + d]);
    out[NEQ - 1] = 0.5 * ((s[NEQ - 1] + po) * vo + (x[NEQ - 1] + px) * vx) -
                   0.5 * lam * (x[NEQ - 1] - s[NEQ - 1]);
  }
}

// Surface contribution of this lane (side, equation group), added into acc.
// All lanes call (shuffles).  Each side evaluates the flux OUT of its own
// element, F_own = lf(own state, other state, own outward normal): no
// left/right selects per point, and the arithmetic of a lane depends only
// on its own element's view of the surface, so a partitioner-flipped
// surface (MC_FLAG_FLIPPED) gives the owned element bit-identical
// contributions without special handling.  The two sides' values are
// negatives of each other up to rounding (the oracle's single flux times
// -/+1 agrees to ~1e-16 relative).
template <class C, int PH, bool kTasks = Tpe<C>::TASKS>
__device__ __forceinline__ void tpe_surface(const double* st, const TpeSide& t, int side, int h,
                                            int nown, const double (&u)[Tpe<C>::WH],
                                            const Params& P, double (&acc)[Tpe<C>::WH],
                                            int grp = 0, double* ws = nullptr) {
  constexpr int NP = C::NP, NEQ = C::NEQ, NEQH = Tpe<C>::NEQH;
  constexpr int H = Tpe<C>::H;
  const double* fphi = st + C::S_FPHI + t.mycode * (C::NQF * C::NPP);
  const double* fw = st + C::S_FW;
  const double sc = -t.scale;
  const int eq0 = h * Tpe<C>::NA;
  double nO[C::DIM];
#pragma unroll
  for (int d = 0; d < C::DIM; ++d) nO[d] = side ? -t.n[d] : t.n[d];
  // H = 1: all traces first, so the coefficients are dead during the flux
  // loop unless the caller still needs them (RK update) — measured +3 % on
  // the surface-only colors of c2.  H = 2: per point, the basis row is read
  // once into registers and used for both the trace and the lift (c3: 0.94
  // vs 0.88 G edges/s for the trace-first form).
  if constexpr (kTasks) {
    // Two lanes per side, fluxes packed as warp tasks: every lane writes its
    // traces to the warp scratch, the warp's (surface, point) fluxes are
    // evaluated once each (SW * NQF tasks over 32 lanes) in the canonical
    // (single-domain) orientation, and each lane lifts its equations with
    // the sign of its canonical side: bit-identical under partitioning.
    constexpr int SW = Tpe<C>::SW, SV = Tpe<C>::SV;
    double* tr = ws + Tpe<C>::X_TR;
    double* fs = ws + Tpe<C>::X_FS;
    double* nrm = ws + Tpe<C>::X_NRM;
    int* flg = reinterpret_cast<int*>(ws + Tpe<C>::X_FLG);
    const int lane = threadIdx.x & 31;
    const bool flip = (t.code & MC_FLAG_FLIPPED) != 0;
    if (side == 0 && h == 0) {
      flg[grp] = t.valid ? (flip ? 2 : 1) : 0;
#pragma unroll
      for (int d = 0; d < C::DIM; ++d) nrm[grp * C::DIM + d] = t.n[d];
    }
#pragma unroll 1
    for (int g = 0; g < C::NQF; ++g) {
#ifndef MC_TRACE_ROW_RELOAD
      // the face-table row once per point, shared by the lane's equations
      // (read per equation it was half of all shared-memory wavefronts of
      // the c4 surface passes, ncu r2c4b)
      double row[C::NPP];
      {
        const double2* r2 = reinterpret_cast<const double2*>(fphi + g * C::NPP);
#pragma unroll
        for (int j = 0; j < C::NPP / 2; ++j) {
          const double2 a = r2[j];
          row[2 * j] = a.x;
          row[2 * j + 1] = a.y;
        }
      }
#endif
#pragma unroll
      for (int k = 0; k < NEQH; ++k) {
        if (k < nown) {
#ifndef MC_TRACE_ROW_RELOAD
          double tv = 0.0;
#pragma unroll
          for (int j = 0; j < NP; ++j) tv = fma(row[j], u[k * NP + j], tv);
          const double v = t.has ? tv : ((t.valid && side) ? P.ff[eq0 + k] : 1.0);
#elif !defined(MC_TRACE_ILP)
          const double v = t.has ? tdot<NP, Tpe<C>::WH>(fphi + g * C::NPP, u, k * NP)
                                 : ((t.valid && side) ? P.ff[eq0 + k] : 1.0);
#else
          // two half-length FMA chains (c4 surface colors -6 % at the
          // 168-register budget of 3 blocks per SM)
          const double v = t.has ? tdot2<NP, Tpe<C>::WH>(fphi + g * C::NPP, u, k * NP)
                                 : ((t.valid && side) ? P.ff[eq0 + k] : 1.0);
#endif
          tr[((g * SW + grp) * 2 + side) * SV + eq0 + k] = v;
        }
      }
    }
    __syncwarp();
#ifdef MC_TASK_UNROLL   // interleaved task pairs: c4 surface colors -4 %
#pragma unroll 2
#endif
    for (int q = lane; q < SW * C::NQF; q += 32) {
      const int g = q / SW, gs = q - g * SW;
      const int f = flg[gs];
      if (f) {
        double sL[NEQ], sR[NEQ], cL[NEQ], cR[NEQ], nn[C::DIM], out[NEQ];
#pragma unroll
        for (int e = 0; e < NEQ; ++e) {
          sL[e] = tr[((g * SW + gs) * 2 + 0) * SV + e];
          sR[e] = tr[((g * SW + gs) * 2 + 1) * SV + e];
        }
        const bool fl = f == 2;
#pragma unroll
        for (int e = 0; e < NEQ; ++e) {
          cL[e] = fl ? sR[e] : sL[e];
          cR[e] = fl ? sL[e] : sR[e];
        }
#pragma unroll
        for (int d = 0; d < C::DIM; ++d) nn[d] = fl ? -nrm[gs * C::DIM + d] : nrm[gs * C::DIM + d];
        Physics<PH, C::DIM, NEQ>::lf(cL, cR, nn, P, out);
#pragma unroll
        for (int e = 0; e < NEQ; ++e) fs[(g * SW + gs) * SV + e] = out[e];
      }
    }
    __syncwarp();
    if (t.owner) {
      // canonical left loses F, canonical right gains it
      const double sc2 = ((side != 0) != flip) ? t.scale : -t.scale;
#pragma unroll 1
      for (int g = 0; g < C::NQF; ++g) {
        const double c = sc2 * fw[g];
#ifndef MC_TRACE_ROW_RELOAD
        double row[C::NPP];
        {
          const double2* r2 = reinterpret_cast<const double2*>(fphi + g * C::NPP);
#pragma unroll
          for (int j = 0; j < C::NPP / 2; ++j) {
            const double2 a = r2[j];
            row[2 * j] = a.x;
            row[2 * j + 1] = a.y;
          }
        }
#pragma unroll
        for (int k = 0; k < NEQH; ++k)
          if (k < nown) {
            const double f = c * fs[(g * SW + grp) * SV + eq0 + k];
#pragma unroll
            for (int j = 0; j < NP; ++j) acc[k * NP + j] = fma(row[j], f, acc[k * NP + j]);
          }
#else
#pragma unroll
        for (int k = 0; k < NEQH; ++k)
          if (k < nown)
            taxpy<NP, Tpe<C>::WH>(fphi + g * C::NPP, c * fs[(g * SW + grp) * SV + eq0 + k], acc,
                                  k * NP);
#endif
      }
    }
    __syncwarp();
  } else if constexpr (H == 1) {
    double trc[C::NQF][NEQH];
#pragma unroll
    for (int g = 0; g < C::NQF; ++g) {
#if defined(MC_H1_ROW_ONCE) && !defined(MC_TRACE_ROW_RELOAD)
      // the table row once per point, not once per equation (opt-in for one
      // lane per side: the fully unrolled point loop then keeps every row
      // live and the RK variants spill 520 bytes at c2's register budget)
      double row[C::NPP];
      {
        const double2* r2 = reinterpret_cast<const double2*>(fphi + g * C::NPP);
#pragma unroll
        for (int j = 0; j < C::NPP / 2; ++j) {
          const double2 a = r2[j];
          row[2 * j] = a.x;
          row[2 * j + 1] = a.y;
        }
      }
#pragma unroll
      for (int k = 0; k < NEQH; ++k) {
        double tv = 0.0;
#pragma unroll
        for (int j = 0; j < NP; ++j) tv = fma(row[j], u[k * NP + j], tv);
        trc[g][k] = t.has ? tv : ((t.valid && side) ? P.ff[k] : 1.0);   // far-field ghost
      }
#else
#pragma unroll
      for (int k = 0; k < NEQH; ++k)
        trc[g][k] = t.has ? tdot<NP, Tpe<C>::WH>(fphi + g * C::NPP, u, k * NP)
                          : ((t.valid && side) ? P.ff[k] : 1.0);   // far-field ghost
#endif
    }
#pragma unroll
    for (int g = 0; g < C::NQF; ++g) {
      double x[NEQ], out[NEQ];
#pragma unroll
      for (int k = 0; k < NEQ; ++k) x[k] = __shfl_xor_sync(kFull, trc[g][k], 1);
#ifdef MC_NO_LF_SHARE
      Physics<PH, C::DIM, NEQ>::lf(trc[g], x, nO, P, out);
#else
      lf_shared<PH, C::DIM, NEQ, 1>(trc[g], x, nO, P, out);
#endif
      if (t.owner) {
        const double c = sc * fw[g];
#if defined(MC_H1_ROW_ONCE) && !defined(MC_TRACE_ROW_RELOAD)
        double row[C::NPP];
        {
          const double2* r2 = reinterpret_cast<const double2*>(fphi + g * C::NPP);
#pragma unroll
          for (int j = 0; j < C::NPP / 2; ++j) {
            const double2 a = r2[j];
            row[2 * j] = a.x;
            row[2 * j + 1] = a.y;
          }
        }
#pragma unroll
        for (int k = 0; k < NEQ; ++k) {
          const double f = c * out[k];
#pragma unroll
          for (int j = 0; j < NP; ++j) acc[k * NP + j] = fma(row[j], f, acc[k * NP + j]);
        }
#else
#pragma unroll
        for (int k = 0; k < NEQ; ++k) taxpy<NP, Tpe<C>::WH>(fphi + g * C::NPP, c * out[k], acc, k * NP);
#endif
      }
    }
  } else {
#pragma unroll 1
    for (int g = 0; g < C::NQF; ++g) {
      double row[C::NPP];
      {
        const double2* r2 = reinterpret_cast<const double2*>(fphi + g * C::NPP);
#pragma unroll
        for (int j = 0; j < C::NPP / 2; ++j) {
          const double2 a = r2[j];
          row[2 * j] = a.x;
          row[2 * j + 1] = a.y;
        }
      }
      double own[NEQH], s[NEQ], x[NEQ], out[NEQ];
#pragma unroll
      for (int k = 0; k < NEQH; ++k) {
        if (t.has) {
          double tr = 0.0;
#pragma unroll
          for (int j = 0; j < NP; ++j) tr = fma(row[j], u[k * NP + j], tr);
          own[k] = tr;
        } else {  // far-field ghost state on physical boundaries
          const int e = (eq0 + k < NEQ) ? eq0 + k : NEQ - 1;
          own[k] = (t.valid && side) ? P.ff[e] : 1.0;
        }
      }
      assemble_state<C>(own, h, s);
#pragma unroll
      for (int k = 0; k < NEQ; ++k) x[k] = __shfl_xor_sync(kFull, s[k], H);
#ifdef MC_NO_LF_SHARE
      Physics<PH, C::DIM, NEQ>::lf(s, x, nO, P, out);
#else
      lf_shared<PH, C::DIM, NEQ, H>(s, x, nO, P, out);
#endif
      if (t.owner) {
        const double c = sc * fw[g];
#pragma unroll
        for (int k = 0; k < NEQH; ++k) {
          if (k < nown) {
            const double f = c * own_part<C>(out, h, k);
#pragma unroll
            for (int j = 0; j < NP; ++j) acc[k * NP + j] = fma(row[j], f, acc[k * NP + j]);
          }
        }
      }
    }
  }
}

// 256-bit accesses (PTX v4.f64; ptxas emits LDG/STG.E.ENL2.256).  CUDA 12.9
// gives double4 only 16-byte alignment, so the C++ type would split them.
// Element blocks are streamed (each read once per launch), so they bypass
// L1 allocation (L1::no_allocate): c3 1.30 -> 1.43 G edges/s, surface-only
// colors 4.5 -> 5.1-5.3 TB/s; c2 neutral to +1 %.  MC_L1_ALLOC restores the
// default caching.
// Tets (c4) measured the other way round once the face-table row was read
// once per point and the colors stopped being side-code sorted: default L1
// allocation 1.483 -> 1.504 G edges/s (colors 2-4 +1.5-3 %), so the policy
// is a template parameter: kL1 = true allocates in L1 (kTpeL1<C>).
// MC_L1_ALLOC / MC_L1_NOALLOC force one policy everywhere.
#define MC_LD_NC_A "ld.global.nc.v4.f64"
#define MC_LD_RW_A "ld.global.v4.f64"
#define MC_LD2_NC_A "ld.global.nc.v2.f64"
#define MC_LD2_RW_A "ld.global.v2.f64"
#define MC_LD_NC_N "ld.global.nc.L1::no_allocate.v4.f64"
#define MC_LD_RW_N "ld.global.L1::no_allocate.v4.f64"
#define MC_LD2_NC_N "ld.global.nc.L1::no_allocate.v2.f64"
#define MC_LD2_RW_N "ld.global.L1::no_allocate.v2.f64"
template <class C>
constexpr bool kTpeL1 =
#if defined(MC_L1_ALLOC)
    true;
#elif defined(MC_L1_NOALLOC)
    false;
#else
    C::DIM == 3;
#endif
template <bool kL1 = false>
__device__ __forceinline__ void ld4_nc(const double* p, double& a, double& b, double& c, double& d) {
  if constexpr (kL1)
    asm(MC_LD_NC_A " {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
  else
    asm(MC_LD_NC_N " {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
template <bool kL1 = false>
__device__ __forceinline__ void ld4(const double* p, double& a, double& b, double& c, double& d) {
  if constexpr (kL1)
    asm(MC_LD_RW_A " {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
  else
    asm(MC_LD_RW_N " {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
template <bool kL1 = false>
__device__ __forceinline__ double2 ld2_nc(const double* p) {
  double2 r;
  if constexpr (kL1)
    asm(MC_LD2_NC_A " {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  else
    asm(MC_LD2_NC_N " {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
template <bool kL1 = false>
__device__ __forceinline__ double2 ld2(const double* p) {
  double2 r;
  if constexpr (kL1)
    asm(MC_LD2_RW_A " {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  else
    asm(MC_LD2_RW_N " {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

// This lane's run of `n` doubles (n <= N): the whole block when H = 1
// (256-bit when N % 4 == 0), its equation group when H = 2 (128-bit pairs).
template <int N, bool kWhole, bool kV4 = kWhole && (N % 4 == 0), bool kL1 = false>
__device__ __forceinline__ void tload(const double* __restrict__ src, int n, double (&dst)[N]) {
  if constexpr (kV4) {   // 32-byte chunks, a 16-byte tail when N % 4 == 2
#pragma unroll
    for (int j = 0; j < N / 4; ++j) {
      if (kWhole || 4 * j + 4 <= n)
        ld4_nc<kL1>(src + 4 * j, dst[4 * j], dst[4 * j + 1], dst[4 * j + 2], dst[4 * j + 3]);
      else
        dst[4 * j] = dst[4 * j + 1] = dst[4 * j + 2] = dst[4 * j + 3] = 0.0;
    }
    if constexpr (N % 4 == 2) {
      if (kWhole || N <= n) {
        const double2 a = ld2_nc<kL1>(src + N - 2);
        dst[N - 2] = a.x;
        dst[N - 1] = a.y;
      } else {
        dst[N - 2] = dst[N - 1] = 0.0;
      }
    }
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      if (kWhole || 2 * j < n) {
        const double2 a = ld2_nc<kL1>(src + 2 * j);
        dst[2 * j] = a.x;
        dst[2 * j + 1] = a.y;
      } else {
        dst[2 * j] = dst[2 * j + 1] = 0.0;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) dst[j] = (kWhole || j < n) ? __ldg(src + j) : 0.0;
  }
}

template <int N, bool kWhole, bool kV4 = kWhole && (N % 4 == 0), bool kL1 = false>
__device__ __forceinline__ void tload_rw(const double* src, int n, double (&dst)[N]) {
  if constexpr (kV4) {
#pragma unroll
    for (int j = 0; j < N / 4; ++j) {
      if (kWhole || 4 * j + 4 <= n)
        ld4<kL1>(src + 4 * j, dst[4 * j], dst[4 * j + 1], dst[4 * j + 2], dst[4 * j + 3]);
      else
        dst[4 * j] = dst[4 * j + 1] = dst[4 * j + 2] = dst[4 * j + 3] = 0.0;
    }
    if constexpr (N % 4 == 2) {
      if (kWhole || N <= n) {
        const double2 a = ld2<kL1>(src + N - 2);
        dst[N - 2] = a.x;
        dst[N - 1] = a.y;
      } else {
        dst[N - 2] = dst[N - 1] = 0.0;
      }
    }
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      if (kWhole || 2 * j < n) {
        const double2 a = ld2<kL1>(src + 2 * j);
        dst[2 * j] = a.x;
        dst[2 * j + 1] = a.y;
      } else {
        dst[2 * j] = dst[2 * j + 1] = 0.0;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) dst[j] = (kWhole || j < n) ? src[j] : 0.0;
  }
}

template <int N, bool kWhole, bool kV4 = kWhole && (N % 4 == 0)>
__device__ __forceinline__ void tstore(double* dst, int n, const double (&src)[N]) {
  if constexpr (kV4) {
#pragma unroll
    for (int j = 0; j < N / 4; ++j)
      if (kWhole || 4 * j + 4 <= n)
        st4(dst + 4 * j, src[4 * j], src[4 * j + 1], src[4 * j + 2], src[4 * j + 3]);
    if constexpr (N % 4 == 2)
      if (kWhole || N <= n)
        *reinterpret_cast<double2*>(dst + N - 2) = make_double2(src[N - 2], src[N - 1]);
  } else if constexpr (N % 2 == 0) {
    double2* d2 = reinterpret_cast<double2*>(dst);
#pragma unroll
    for (int j = 0; j < N / 2; ++j)
      if (kWhole || 2 * j < n) d2[j] = make_double2(src[2 * j], src[2 * j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (kWhole || j < n) dst[j] = src[j];
  }
}

// fp32 state storage (DGOperator(state="f32"); the north star's "1e-5
// (fp32)" tolerance): element blocks of floats, converted to double on load
// and rounded back on store; all arithmetic stays fp64.  Runs are 16-byte
// aligned (float strides are multiples of 4), moved as 128-bit accesses.
__device__ __forceinline__ void ld4f(const float* p, bool nc, double& a, double& b, double& c,
                                     double& d) {
  float x, y, z, w;
  if (nc)
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "l"(p));
  else
    asm("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "l"(p));
  a = x;
  b = y;
  c = z;
  d = w;
}

template <int N, bool kWhole>
__device__ __forceinline__ void fload(const float* src, int n, double (&dst)[N], bool nc) {
#pragma unroll
  for (int j = 0; j < N / 4; ++j) {
    if (kWhole || 4 * j + 4 <= n)
      ld4f(src + 4 * j, nc, dst[4 * j], dst[4 * j + 1], dst[4 * j + 2], dst[4 * j + 3]);
    else
      dst[4 * j] = dst[4 * j + 1] = dst[4 * j + 2] = dst[4 * j + 3] = 0.0;
  }
#pragma unroll
  for (int j = N / 4 * 4; j < N; ++j) dst[j] = (kWhole || j < n) ? double(src[j]) : 0.0;
}

template <int N, bool kWhole>
__device__ __forceinline__ void fstore(float* dst, int n, const double (&src)[N]) {
#pragma unroll
  for (int j = 0; j < N / 4; ++j)
    if (kWhole || 4 * j + 4 <= n)
      *reinterpret_cast<float4*>(dst + 4 * j) =
          make_float4(__double2float_rn(src[4 * j]), __double2float_rn(src[4 * j + 1]),
                      __double2float_rn(src[4 * j + 2]), __double2float_rn(src[4 * j + 3]));
#pragma unroll
  for (int j = N / 4 * 4; j < N; ++j)
    if (kWhole || j < n) dst[j] = __double2float_rn(src[j]);
}

// fp32 runs that are only 8-byte aligned (two lanes per side with an odd
// basis size, e.g. quads / hybrid meshes at p = 2: lane 1 starts 18 floats
// into the block): 64-bit float pairs instead of 128-bit quads
template <int N, bool kWhole>
__device__ __forceinline__ void fload2(const float* src, int n, double (&dst)[N], bool nc) {
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    if (kWhole || 2 * j + 2 <= n) {
      float x, y;
      if (nc)
        asm("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y)
            : "l"(src + 2 * j));
      else
        asm("ld.global.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y)
            : "l"(src + 2 * j));
      dst[2 * j] = x;
      dst[2 * j + 1] = y;
    } else {
      dst[2 * j] = dst[2 * j + 1] = 0.0;
    }
  }
  if constexpr (N % 2) dst[N - 1] = (kWhole || N <= n) ? double(src[N - 1]) : 0.0;
}

template <int N, bool kWhole>
__device__ __forceinline__ void fstore2(float* dst, int n, const double (&src)[N]) {
#pragma unroll
  for (int j = 0; j < N / 2; ++j)
    if (kWhole || 2 * j + 2 <= n)
      *reinterpret_cast<float2*>(dst + 2 * j) =
          make_float2(__double2float_rn(src[2 * j]), __double2float_rn(src[2 * j + 1]));
  if constexpr (N % 2)
    if (kWhole || N <= n) dst[N - 1] = __double2float_rn(src[N - 1]);
}

// state-type dispatch: S = double (the default) or float
template <int N, bool kWhole, bool kV4, bool kL1 = false>
__device__ __forceinline__ void sload(const double* src, int n, double (&dst)[N]) {
  tload<N, kWhole, kV4, kL1>(src, n, dst);
}
template <int N, bool kWhole, bool kV4, bool kL1 = false>
__device__ __forceinline__ void sload(const float* src, int n, double (&dst)[N]) {
  if constexpr (kWhole || kV4) fload<N, kWhole>(src, n, dst, true);
  else fload2<N, kWhole>(src, n, dst, true);
}
template <int N, bool kWhole, bool kV4, bool kL1 = false>
__device__ __forceinline__ void sload_rw(const double* src, int n, double (&dst)[N]) {
  tload_rw<N, kWhole, kV4, kL1>(src, n, dst);
}
template <int N, bool kWhole, bool kV4, bool kL1 = false>
__device__ __forceinline__ void sload_rw(const float* src, int n, double (&dst)[N]) {
  if constexpr (kWhole || kV4) fload<N, kWhole>(src, n, dst, false);
  else fload2<N, kWhole>(src, n, dst, false);
}
template <int N, bool kWhole, bool kV4>
__device__ __forceinline__ void sstore(double* dst, int n, const double (&src)[N]) {
  tstore<N, kWhole, kV4>(dst, n, src);
}
template <int N, bool kWhole, bool kV4>
__device__ __forceinline__ void sstore(float* dst, int n, const double (&src)[N]) {
  if constexpr (kWhole || kV4) fstore<N, kWhole>(dst, n, src);
  else fstore2<N, kWhole>(dst, n, src);
}

template <class C>
__device__ __forceinline__ void tpe_stage(const double* __restrict__ g, double* s) {
  stage_tables<C>(g, s);
}

// ------------------------------------------------------------- kernels
#ifndef MC_TPE_MINB_SURF
#define MC_TPE_MINB_SURF 3
#endif
#ifndef MC_TPE_MINB_RK
#define MC_TPE_MINB_RK 3
#endif
// two lanes per side: blocks per SM of the surface-only (3: c4 colors 2-3
// 3.98 -> 4.40 TB/s, c3 +1 %), first-touch (tets 3: +5 %; quads keep 2:
// -18 %) and last-touch passes; each variant gets its own resident grid
#ifndef MC_TASKS_MINB_SURF
#define MC_TASKS_MINB_SURF 3
#endif
#ifndef MC_TPE_MINB_RK2
#define MC_TPE_MINB_RK2 2
#endif
#ifndef MC_TPE_MINB_VOL
#define MC_TPE_MINB_VOL 0   // 0: Tpe<C>::MINB
#endif
#ifndef MC_TPE_MINB_VOL2
// two lanes per side, first-touch passes (tets): 2 blocks per SM (255
// registers, no spills) since the face-table-row change; 3 blocks (168
// registers, 104-byte spills) measured 1.414 vs 1.447 G edges/s on c4
#define MC_TPE_MINB_VOL2 2
#endif

// surface-flux scheme per kernel variant: warp flux tasks (Tpe::TASKS /
// TASKS_SURF) or each lane's own flux; MC_RK_NO_TASKS / MC_VOL_NO_TASKS
// switch the last-touch / first-touch variants to per-lane fluxes (A/B)
template <class T, bool kRK, bool kVol>
constexpr bool kVariantTasks =
#if defined(MC_VOL_NO_TASKS)
    kVol ? false :
#endif
#if defined(MC_RK_NO_TASKS)
    (kRK && !kVol) ? false :
#endif
    (kVol ? T::TASKS : T::TASKS_SURF);

struct TpeLane {
  int lane, side, h, grp, nown, eq0;
};

template <class C>
__device__ __forceinline__ TpeLane tpe_lane() {
  constexpr int H = Tpe<C>::H;
  TpeLane L;
  L.lane = threadIdx.x & 31;
  L.grp = L.lane / (2 * H);
  L.side = (L.lane / H) & 1;
  L.h = L.lane % H;
  L.eq0 = L.h * Tpe<C>::NA;
  L.nown = (L.h == 0) ? Tpe<C>::NA : Tpe<C>::NEQH;
  return L;
}

// kVol: the color contains first touches (volume fused); kRK: the color
// contains last touches of an RK stage (update fused).  The host picks the
// variant per color launch so surface-only passes carry no volume code.
template <class C, int PH, bool kRK, bool kVol, class S = double>
__global__ void __launch_bounds__(Tpe<C>::THREADS,
                                  Tpe<C>::H == 2
                                      ? ((!kVol && !kRK) ? MC_TASKS_MINB_SURF
                                         : kVol ? (C::DIM == 3 ? MC_TPE_MINB_VOL2 : 2)
                                                : MC_TPE_MINB_RK2)
                                  : kVol ? (MC_TPE_MINB_VOL ? MC_TPE_MINB_VOL : Tpe<C>::MINB)
                                  : (kRK ? MC_TPE_MINB_RK : MC_TPE_MINB_SURF))
k_tpe_colored(View v, S* __restrict__ U, S* __restrict__ R, RK rk, int64_t begin,
              int64_t end) {
  S* const U0 = static_cast<S*>(rk.U0);
  using T = Tpe<C>;
  constexpr int WH = T::WH;
  constexpr bool kWhole = T::H == 1;
  extern __shared__ double sts[];
  tpe_stage<C>(v.tables, sts);
  const double* st = sts;
  double* ws = sts + C::S_TOTAL + (threadIdx.x >> 5) * T::X_SIZE;   // TASKS scratch
  const TpeLane ln = tpe_lane<C>();
  const int n = ln.nown * C::NP;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
#ifndef MC_NO_E_PREFETCH
  const int32_t* eidx = ln.side ? v.right : v.left;
  int e_next = -1;
#ifdef MC_CODE_PREFETCH
  uint32_t c_next = 0;   // the surface code word one tile ahead as well
#endif
  {
    const int64_t s0 = begin + warp * T::SW + ln.grp;
    if (s0 < end) e_next = __ldg(eidx + s0);
#ifdef MC_CODE_PREFETCH
    if (s0 < end) c_next = __ldg(v.code + s0);
#endif
  }
#endif
  for (int64_t tile = begin + warp * T::SW; tile < end; tile += nwarp * T::SW) {
    const int64_t s = tile + ln.grp;
#ifndef MC_NO_E_PREFETCH
#ifdef MC_CODE_PREFETCH
    const TpeSide t = tpe_side_pre<C>(v, s, end, ln.side, e_next, &c_next);
#else
    const TpeSide t = tpe_side_pre<C>(v, s, end, ln.side, e_next);
#endif
    {
      const int64_t sn = s + nwarp * T::SW;
      e_next = sn < end ? __ldg(eidx + sn) : -1;
#ifdef MC_CODE_PREFETCH
      c_next = sn < end ? __ldg(v.code + sn) : 0u;
#endif
    }
#else
    const TpeSide t = tpe_side<C>(v, s, end, ln.side);
#endif
    const bool first = kVol && t.owner && (t.code & (ln.side ? MC_FLAG_R_FIRST : MC_FLAG_L_FIRST));
    const bool last = kRK && t.owner && (t.code & (ln.side ? MC_FLAG_R_LAST : MC_FLAG_L_LAST));
    const int64_t off = int64_t(t.has ? t.e : 0) * v.stride + ln.eq0 * C::NP;
#ifdef MC_U0_PREFETCH
    // last-touch passes: pull the RK base block into L1 now, read it at the end
    if (kRK && last && rk.a != 0.0) {
      const char* p0 = reinterpret_cast<const char*>(U0 + off);
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p0));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p0 + 128));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p0 + n * sizeof(S) - 1));
    }
#endif
    double u[WH], acc[WH];
    if (t.has) sload<WH, kWhole, T::V4, kTpeL1<C>>(U + off, n, u);
    else {
#pragma unroll
      for (int j = 0; j < WH; ++j) u[j] = 0.0;
    }
    if constexpr (kVol && kVolBal<C>) {   // lane 0: the last equation in its spare slot
      if (ln.h == 0 && first)
        sload<C::NP, true, false>(U + int64_t(t.e) * v.stride + (C::NEQ - 1) * C::NP, C::NP,
                                  bal_slot<C>(u));
    }
    // first-touch passes: the volume integral first, then the residual
    // blocks of the sides touched before (acc is not live during the volume)
    if (kVol || !(t.owner && !first)) {
#pragma unroll
      for (int j = 0; j < WH; ++j) acc[j] = 0.0;
    } else {
      sload_rw<WH, kWhole, T::V4, kTpeL1<C>>(R + off, n, acc);
    }
    if constexpr (kVol) {
      const double* jp = v.jinv + int64_t(first ? t.e : 0) * (C::DIM * C::DIM);
      int ek = 0;
      if constexpr (C::KIND == HYB) ek = first ? __ldg(v.ekind + t.e) : 0;
      if constexpr (T::H == 1) {
        if (first) tpe_volume<C, PH>(st, u, jp, 0, ln.nown, true, v.prm, acc, ek);
      } else if (__any_sync(kFull, first)) {   // the whole warp takes part in the shuffles
#ifndef MC_NO_JINV_ASYNC
        // the Jacobian through the (idle) flux-task scratch, one slot per side
        // (c4 color 1 +2 % at 2 blocks/SM: the lift no longer waits on its loads)
        double* jst = kVariantTasks<T, kRK, kVol>
                          ? ws + (ln.lane / T::H) * (C::DIM * C::DIM) : nullptr;
#else
        double* jst = nullptr;
#endif
        tpe_volume<C, PH>(st, u, jp, ln.h, ln.nown, first, v.prm, acc, ek, jst);
      }
      if (t.owner && !first) sload_rw<WH, kWhole, T::V4, kTpeL1<C>>(R + off, n, acc);
    }
    tpe_surface<C, PH, kVariantTasks<T, kRK, kVol>>(st, t, ln.side, ln.h, ln.nown, u, v.prm, acc,
                                                     ln.grp, ws);
    if (t.owner) {
      if (last) {
#ifdef MC_RK_RELOAD_U
        // re-read the element's own block (L2) instead of keeping u live
        // through the surface work (fewer registers in the last-touch pass)
        if constexpr (kRK && !kVol) sload<WH, kWhole, T::V4, kTpeL1<C>>(U + off, n, u);
#endif
        if (rk.save_u0) sstore<WH, kWhole, T::V4>(U0 + off, n, u);
        if (rk.a != 0.0) {
          double u0[WH];
          sload<WH, kWhole, T::V4, kTpeL1<C>>(U0 + off, n, u0);
#pragma unroll
          for (int j = 0; j < WH; ++j) acc[j] = rk.a * u0[j] + rk.b * fma(rk.dt, acc[j], u[j]);
        } else {
#pragma unroll
          for (int j = 0; j < WH; ++j) acc[j] = rk.b * fma(rk.dt, acc[j], u[j]);
        }
        sstore<WH, kWhole, T::V4>(U + off, n, acc);
        if (v.send_slot) {
          const int sl = __ldg(v.send_slot + t.e);
          if (sl >= 0)
            sstore<WH, kWhole, T::V4>(static_cast<S*>(v.send_buf) + int64_t(sl) * v.stride + ln.eq0 * C::NP, n, acc);
        }
        if (v.push_ptr) {   // peer push: the new block into the peers' ghost rows
          const int64_t k1 = __ldg(v.push_ptr + t.e + 1);
          for (int64_t k = __ldg(v.push_ptr + t.e); k < k1; ++k) {
            S* d = reinterpret_cast<S*>(__ldg(v.push_dst + k)) + v.push_shift + ln.eq0 * C::NP;
            sstore<WH, kWhole, T::V4>(d, n, acc);
          }
        }
      } else {
        sstore<WH, kWhole, T::V4>(R + off, n, acc);
      }
    }
  }
}

template <class C, int PH, bool kAtomic>
__global__ void __launch_bounds__(Tpe<C>::THREADS, Tpe<C>::MINB)
k_tpe_uncolored(View v, const double* __restrict__ U, double* __restrict__ out) {
  using T = Tpe<C>;
  constexpr int WH = T::WH;
  constexpr bool kWhole = T::H == 1;
  extern __shared__ double st[];
  tpe_stage<C>(v.tables, st);
  double* ws = st + C::S_TOTAL + (threadIdx.x >> 5) * T::X_SIZE;   // TASKS scratch
  const TpeLane ln = tpe_lane<C>();
  const int n = ln.nown * C::NP;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t end = v.n_surfaces;
  for (int64_t tile = warp * T::SW; tile < end; tile += nwarp * T::SW) {
    const int64_t s = tile + ln.grp;
    const TpeSide t = tpe_side<C>(v, s, end, ln.side);
    double u[WH], acc[WH];
    if (t.has) tload<WH, kWhole, T::V4>(U + int64_t(t.e) * v.stride + ln.eq0 * C::NP, n, u);
    else {
#pragma unroll
      for (int j = 0; j < WH; ++j) u[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < WH; ++j) acc[j] = 0.0;
    tpe_surface<C, PH>(st, t, ln.side, ln.h, ln.nown, u, v.prm, acc, ln.grp, ws);
    if (kAtomic) {
      if (t.owner) {
        double* dst = out + int64_t(t.e) * v.stride + ln.eq0 * C::NP;
#pragma unroll
        for (int j = 0; j < WH; ++j)
          if (kWhole || j < n) atomicAdd(dst + j, acc[j]);
      }
    } else if (t.valid) {
      if (!t.owner) {
#pragma unroll
        for (int j = 0; j < WH; ++j) acc[j] = 0.0;
      }
      tstore<WH, kWhole, T::V4>(out + (2 * s + ln.side) * v.stride + ln.eq0 * C::NP, n, acc);
    }
  }
}

// Volume integral for all owned elements (unfused strategies): H lanes per
// element, 32/H elements per warp.
template <class C, int PH>
__global__ void __launch_bounds__(Tpe<C>::THREADS, Tpe<C>::MINB)
k_tpe_volume(View v, const double* __restrict__ U, double* __restrict__ R) {
  using T = Tpe<C>;
  constexpr int WH = T::WH, H = T::H;
  constexpr bool kWhole = H == 1;
  extern __shared__ double st[];
  tpe_stage<C>(v.tables, st);
  const int lane = threadIdx.x & 31, h = lane % H;
  const int nown = (h == 0) ? T::NA : T::NEQH, eq0 = h * T::NA, n = nown * C::NP;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t tile = warp * (32 / H); tile < v.n_elements; tile += nwarp * (32 / H)) {
    const int64_t e = tile + lane / H;
    const bool has = e < v.n_elements;
    const int64_t off = (has ? e : 0) * v.stride + eq0 * C::NP;
    double u[WH], acc[WH];
    if (has) tload<WH, kWhole, T::V4>(U + off, n, u);
    else {
#pragma unroll
      for (int j = 0; j < WH; ++j) u[j] = 0.0;
    }
    if constexpr (kVolBal<C>) {
      if (h == 0 && has)
        tload<C::NP, true, false>(U + e * v.stride + (C::NEQ - 1) * C::NP, C::NP, bal_slot<C>(u));
    }
#pragma unroll
    for (int j = 0; j < WH; ++j) acc[j] = 0.0;
    int ek = 0;
    if constexpr (C::KIND == HYB) ek = has ? __ldg(v.ekind + e) : 0;
    tpe_volume<C, PH>(st, u, v.jinv + (has ? e : 0) * (C::DIM * C::DIM), h, nown, has, v.prm,
                      acc, ek);
    if (has) tstore<WH, kWhole, T::V4>(R + off, n, acc);
  }
}

// Write the padded table layout (what tpe_stage puts in shared memory) to
// global memory once per operator (kept for experiments reading tables via L1).
template <class C>
__global__ void k_stage_global(const double* __restrict__ g, double* out) {
  extern __shared__ double sts[];
  stage_tables<C>(g, sts);
  for (int i = threadIdx.x; i < C::S_TOTAL; i += blockDim.x) out[i] = sts[i];
}

}  // namespace mcdg
