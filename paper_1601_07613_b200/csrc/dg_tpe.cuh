// Thread-per-element-side DG kernels for small element blocks
// (N_eq * N_p <= 24 doubles: c1 advection p=1, c2 Euler p=2 on triangles,
// Euler p=1 on quads, ...).
//
// Each lane owns a WHOLE element block in registers: lanes (2i, 2i+1) are
// the left / right side of surface i, 16 surfaces per warp.  A lane loads
// its element's coefficients with 16-byte loads (high memory-level
// parallelism: the whole block is in flight at once), evaluates its own
// traces, swaps them with its partner through one shuffle per equation,
// evaluates the Lax-Friedrichs flux (both partners compute the same value),
// lifts it into its own residual block and stores.  In the first-touch pass
// it also evaluates the element's volume integral (one flux per volume
// point, no redundancy).  Reference-element tables live in shared memory
// and are read either as warp-wide broadcasts (volume tables) or per lane
// (face tables, indexed by the side code).  No shared-memory staging of
// per-element data at all — this is what the smem-bound group kernel
// (dg_kernels.cuh) cannot avoid.
//
// Same accumulation order per element as Algorithm 1 and the oracle:
// volume, then colors 1..n; within a surface the quadrature points in order.
#pragma once

#include "dg_kernels.cuh"

namespace mcdg {

template <class C>
struct Tpe {
  static constexpr bool OK = C::NEQ * C::NP <= 24;
  static constexpr int W = C::NEQ * C::NP;
  static constexpr int THREADS = 128;
#ifdef MC_MINB_TPE
  static constexpr int MINB = MC_MINB_TPE;
#else
  static constexpr int MINB = (C::NEQ * C::NP > 16) ? 3 : 4;
#endif
  static constexpr int SMEM = C::S_TOTAL * 8;
};

// sum_j row[j] * u[off + j]
template <int NP, int W>
__device__ __forceinline__ double tdot(const double* row, const double (&u)[W], int off) {
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

template <int NP, int W>
__device__ __forceinline__ void taxpy(const double* row, double f, double (&acc)[W], int off) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int j = 0; j < NP / 2; ++j) {
    const double2 a = r2[j];
    acc[off + 2 * j] = fma(a.x, f, acc[off + 2 * j]);
    acc[off + 2 * j + 1] = fma(a.y, f, acc[off + 2 * j + 1]);
  }
  if constexpr (NP % 2) acc[off + NP - 1] = fma(row[NP - 1], f, acc[off + NP - 1]);
}

// Volume integral of one element (this lane), added into acc.
template <class C, int PH>
__device__ __forceinline__ void tpe_volume(const double* st, const double (&u)[Tpe<C>::W],
                                           const double* __restrict__ jinv_e, const Params& P,
                                           double (&acc)[Tpe<C>::W]) {
  constexpr int W = Tpe<C>::W, NP = C::NP, NEQ = C::NEQ, DIM = C::DIM;
  const double* vphi = st + C::S_VPHI;
  const double* vdphi = st + C::S_VDPHI;
  const double* vw = st + C::S_VW;
  double ji[DIM * DIM];
#pragma unroll
  for (int k = 0; k < DIM * DIM; ++k) ji[k] = __ldg(jinv_e + k);
#pragma unroll 1
  for (int q = 0; q < C::NQV; ++q) {
    double s[NEQ];
#pragma unroll
    for (int k = 0; k < NEQ; ++k) s[k] = tdot<NP, W>(vphi + q * C::NPP, u, k * NP);
    const double w = vw[q];
    if constexpr (PH == EULER) {
      const double inv = 1.0 / s[0];
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
        taxpy<NP, W>(dp, w * (s[0] * ut), acc, 0);
#pragma unroll
        for (int d = 0; d < DIM; ++d)
          taxpy<NP, W>(dp, w * (s[1 + d] * ut + p * ji[r * DIM + d]), acc, (1 + d) * NP);
        taxpy<NP, W>(dp, w * ((s[NEQ - 1] + p) * ut), acc, (NEQ - 1) * NP);
      }
    } else {
#pragma unroll
      for (int r = 0; r < DIM; ++r) {
        double a = ji[r * DIM + 0] * P.vel[0] + ji[r * DIM + 1] * P.vel[1];
        if (DIM == 3) a += ji[r * DIM + 2] * P.vel[2];
        taxpy<NP, W>(vdphi + (r * C::NQV + q) * C::NPP, w * (a * s[0]), acc, 0);
      }
    }
  }
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
  t.e = side ? R : L;
  t.has = t.valid && t.e >= 0;
  t.owner = t.has && !(side && (t.code & MC_FLAG_R_GHOST));
  t.mycode = side ? int((t.code >> 6) & 63u) : int(t.code & 63u);
  return t;
}

// Surface contribution of this lane's side, added into acc.  All lanes call.
template <class C, int PH>
__device__ __forceinline__ void tpe_surface(const double* st, const TpeSide& t, int side,
                                            const double (&u)[Tpe<C>::W], const Params& P,
                                            double (&acc)[Tpe<C>::W]) {
  constexpr int W = Tpe<C>::W, NP = C::NP, NEQ = C::NEQ;
  const double* fphi = st + C::S_FPHI + t.mycode * (C::NQF * C::NPP);
  const double* fw = st + C::S_FW;
  const double sc = side ? t.scale : -t.scale;
#pragma unroll 1
  for (int g = 0; g < C::NQF; ++g) {
    double own[NEQ], sL[NEQ], sR[NEQ], out[NEQ], row[C::NPP];
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
      if (t.has) {
        double tr = 0.0;
#pragma unroll
        for (int j = 0; j < NP; ++j) tr = fma(row[j], u[k * NP + j], tr);
        own[k] = tr;
      } else {
        own[k] = (t.valid && side) ? P.ff[k] : 0.0;   // far-field ghost
      }
      const double other = __shfl_xor_sync(kFull, own[k], 1);
      sL[k] = side ? other : own[k];
      sR[k] = side ? own[k] : other;
    }
    // canonical (single-domain) orientation for partitioner-flipped surfaces,
    // through ONE call site so the arithmetic is bit-identical to 1 domain
    const bool flip = (t.code & MC_FLAG_FLIPPED) != 0;
    double cL[NEQ], cR[NEQ], nn[C::DIM];
#pragma unroll
    for (int k = 0; k < NEQ; ++k) {
      cL[k] = flip ? sR[k] : sL[k];
      cR[k] = flip ? sL[k] : sR[k];
    }
#pragma unroll
    for (int d = 0; d < C::DIM; ++d) nn[d] = flip ? -t.n[d] : t.n[d];
    Physics<PH, C::DIM, NEQ>::lf(cL, cR, nn, P, out);
    double c = sc * fw[g];
    if (flip) c = -c;
    if (t.owner) {
#pragma unroll
      for (int k = 0; k < NEQ; ++k) {
        const double f = c * out[k];
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[k * NP + j] = fma(row[j], f, acc[k * NP + j]);
      }
    }
  }
}

// Whole-block loads/stores.  Blocks are 32-byte aligned (stride padded to
// 4 doubles), so W % 4 == 0 blocks move as 256-bit accesses
// (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a): one full 32-byte sector per
// lane per instruction, half the L1 wavefronts of 128-bit accesses.
// 256-bit accesses (PTX v4.f64; ptxas emits LDG/STG.E.ENL2.256).  CUDA 12.9
// gives double4 only 16-byte alignment, so the C++ type would split them.
__device__ __forceinline__ void ld4_nc(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void ld4(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

template <int W>
__device__ __forceinline__ void tload(const double* __restrict__ src, double (&dst)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int j = 0; j < W / 4; ++j)
      ld4_nc(src + 4 * j, dst[4 * j], dst[4 * j + 1], dst[4 * j + 2], dst[4 * j + 3]);
  } else {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int j = 0; j < W / 2; ++j) {
      const double2 a = __ldg(s2 + j);
      dst[2 * j] = a.x;
      dst[2 * j + 1] = a.y;
    }
    if constexpr (W % 2) dst[W - 1] = __ldg(src + W - 1);
  }
}

template <int W>
__device__ __forceinline__ void tload_rw(const double* src, double (&dst)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int j = 0; j < W / 4; ++j)
      ld4(src + 4 * j, dst[4 * j], dst[4 * j + 1], dst[4 * j + 2], dst[4 * j + 3]);
  } else {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int j = 0; j < W / 2; ++j) {
      const double2 a = s2[j];
      dst[2 * j] = a.x;
      dst[2 * j + 1] = a.y;
    }
    if constexpr (W % 2) dst[W - 1] = src[W - 1];
  }
}

template <int W>
__device__ __forceinline__ void tstore(double* dst, const double (&src)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int j = 0; j < W / 4; ++j)
      st4(dst + 4 * j, src[4 * j], src[4 * j + 1], src[4 * j + 2], src[4 * j + 3]);
  } else {
    double2* d2 = reinterpret_cast<double2*>(dst);
#pragma unroll
    for (int j = 0; j < W / 2; ++j) d2[j] = make_double2(src[2 * j], src[2 * j + 1]);
    if constexpr (W % 2) dst[W - 1] = src[W - 1];
  }
}

template <class C>
__device__ __forceinline__ void tpe_stage(const double* __restrict__ g, double* s) {
  stage_tables<C>(g, s);
}

// ------------------------------------------------------------- kernels
// L2 prefetch of a whole element block through the TMA engine (one
// instruction per block; the data lands in L2 while the current tile
// computes, so the next tile's loads hit L2 instead of waiting on HBM).
__device__ __forceinline__ void prefetch_l2(const double* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// kVol: the color contains first touches (volume fused); kRK: the color
// contains last touches of an RK stage (update fused).  The host picks the
// variant per color launch so surface-only passes carry no volume code.
#ifndef MC_TPE_GLOBAL_TABLES
#define MC_TPE_GLOBAL_TABLES 0
#endif
#ifndef MC_TPE_MINB_SURF
#define MC_TPE_MINB_SURF 3
#endif
template <class C, int PH, bool kRK, bool kVol>
__global__ void __launch_bounds__(Tpe<C>::THREADS, kVol ? Tpe<C>::MINB : MC_TPE_MINB_SURF)
k_tpe_colored(View v, double* __restrict__ U, double* __restrict__ R, RK rk, int64_t begin,
              int64_t end) {
  constexpr int W = Tpe<C>::W;
#if MC_TPE_GLOBAL_TABLES
  const double* st = v.ptables;          // 4-30 KB, stays L1/L2 resident
#else
  extern __shared__ double sts[];
  tpe_stage<C>(v.tables, sts);
  const double* st = sts;
#endif
  const int lane = threadIdx.x & 31, side = lane & 1;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
#ifdef MC_TPE_PREFETCH
  const uint32_t blk = uint32_t(v.stride * 8);
#endif
  for (int64_t tile = begin + warp * 16; tile < end; tile += nwarp * 16) {
    const int64_t s = tile + (lane >> 1);
#ifdef MC_TPE_PREFETCH
    {  // prefetch the next tile of this warp into L2
      const int64_t sn = s + nwarp * 16;
      if (sn < end) {
        const int en = side ? __ldg(v.right + sn) : __ldg(v.left + sn);
        if (en >= 0) {
          prefetch_l2(U + int64_t(en) * v.stride, blk);
          if (!kVol && en < v.n_elements) prefetch_l2(R + int64_t(en) * v.stride, blk);
          if (kRK && rk.a != 0.0 && en < v.n_elements) prefetch_l2(rk.U0 + int64_t(en) * v.stride, blk);
        }
      }
    }
#endif
    const TpeSide t = tpe_side<C>(v, s, end, side);
    const bool first = kVol && t.owner && (t.code & (side ? MC_FLAG_R_FIRST : MC_FLAG_L_FIRST));
    const bool last = kRK && t.owner && (t.code & (side ? MC_FLAG_R_LAST : MC_FLAG_L_LAST));
    const int64_t off = int64_t(t.has ? t.e : 0) * v.stride;
    double u[W], acc[W];
    if (t.has) tload<W>(U + off, u);
    else {
#pragma unroll
      for (int j = 0; j < W; ++j) u[j] = 0.0;
    }
    if (t.owner && !first) tload_rw<W>(R + off, acc);
    else {
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = 0.0;
    }
    if constexpr (kVol) {
      if (first) tpe_volume<C, PH>(st, u, v.jinv + int64_t(t.e) * (C::DIM * C::DIM), v.prm, acc);
    }
    tpe_surface<C, PH>(st, t, side, u, v.prm, acc);
    if (t.owner) {
      if (last) {
        if (rk.save_u0) tstore<W>(rk.U0 + off, u);
        if (rk.a != 0.0) {
          double u0[W];
          tload<W>(rk.U0 + off, u0);
#pragma unroll
          for (int j = 0; j < W; ++j) acc[j] = rk.a * u0[j] + rk.b * fma(rk.dt, acc[j], u[j]);
        } else {
#pragma unroll
          for (int j = 0; j < W; ++j) acc[j] = rk.b * fma(rk.dt, acc[j], u[j]);
        }
        tstore<W>(U + off, acc);
      } else {
        tstore<W>(R + off, acc);
      }
    }
  }
}

template <class C, int PH, bool kAtomic>
__global__ void __launch_bounds__(Tpe<C>::THREADS, Tpe<C>::MINB)
k_tpe_uncolored(View v, const double* __restrict__ U, double* __restrict__ out) {
  constexpr int W = Tpe<C>::W;
  extern __shared__ double st[];
  tpe_stage<C>(v.tables, st);
  const int lane = threadIdx.x & 31, side = lane & 1;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t end = v.n_surfaces;
  for (int64_t tile = warp * 16; tile < end; tile += nwarp * 16) {
    const int64_t s = tile + (lane >> 1);
    const TpeSide t = tpe_side<C>(v, s, end, side);
    double u[W], acc[W];
    if (t.has) tload<W>(U + int64_t(t.e) * v.stride, u);
    else {
#pragma unroll
      for (int j = 0; j < W; ++j) u[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] = 0.0;
    tpe_surface<C, PH>(st, t, side, u, v.prm, acc);
    if (kAtomic) {
      if (t.owner) {
        double* dst = out + int64_t(t.e) * v.stride;
#pragma unroll
        for (int j = 0; j < W; ++j) atomicAdd(dst + j, acc[j]);
      }
    } else if (t.valid) {
      if (!t.owner) {
#pragma unroll
        for (int j = 0; j < W; ++j) acc[j] = 0.0;
      }
      tstore<W>(out + (2 * s + side) * v.stride, acc);
    }
  }
}

template <class C, int PH>
__global__ void __launch_bounds__(Tpe<C>::THREADS, Tpe<C>::MINB)
k_tpe_volume(View v, const double* __restrict__ U, double* __restrict__ R) {
  constexpr int W = Tpe<C>::W;
  extern __shared__ double st[];
  tpe_stage<C>(v.tables, st);
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < v.n_elements;
       e += int64_t(gridDim.x) * blockDim.x) {
    double u[W], acc[W];
    tload<W>(U + e * v.stride, u);
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] = 0.0;
    tpe_volume<C, PH>(st, u, v.jinv + e * (C::DIM * C::DIM), v.prm, acc);
    tstore<W>(R + e * v.stride, acc);
  }
}

// Write the padded table layout (what tpe_stage puts in shared memory) to
// global memory once per operator; kernels may read it through L1.
template <class C>
__global__ void k_stage_global(const double* __restrict__ g, double* out) {
  extern __shared__ double sts[];
  stage_tables<C>(g, sts);
  for (int i = threadIdx.x; i < C::S_TOTAL; i += blockDim.x) out[i] = sts[i];
}

}  // namespace mcdg
