// Type-erased launchers for one (kind, physics, degree) instantiation.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dg_kernels.cuh"
#include "dg_tpe.cuh"

namespace mcdg {

struct Ops {
  int dim, neq, np, nqf, nqv, ncodes, table_size;
  int threads;                                     // block size of the task kernels
  int spw;                                         // surfaces per warp
  int grid_colored, grid_volume, grid_uncolored;   // resident-grid sizes
  // per colored-kernel variant, index (rk-update ? 2 : 0) | (volume ? 1 : 0):
  // each variant has its own register budget, so its own resident grid
  int grid_var[4];
  // U / R point to element blocks of the state type: double, or float when
  // f32 (fp32 state storage, register kernels only)
  cudaError_t (*colored)(const View&, void* U, void* R, const RK* rk, int64_t b,
                         int64_t e, int grid, cudaStream_t s, bool has_first, bool has_last,
                         bool f32);
  cudaError_t (*volume)(const View&, const double* U, double* R, int grid, cudaStream_t s);
  cudaError_t (*uncolored)(const View&, const double* U, double* out, bool atomic, int grid,
                           cudaStream_t s);
  cudaError_t (*gather)(const View&, const double* buf, double* R, int cap, cudaStream_t s);
  cudaError_t (*init)(Ops* self);   // occupancy queries, smem opt-in
  int stable_size;                  // doubles of the padded table layout
  cudaError_t (*stage_global)(const double* tables, double* out, cudaStream_t s);
  // copy the volume part of the padded tables into this configuration's
  // constant-memory array (c_voltab)
  cudaError_t (*upload_const)(const double* ptables_dev);
  int npl;                          // P_{p-1} modes of the factored projection
  int p1proj;                       // the register kernels use it (Cfg::P1PROJ)
  int tpe;                          // register kernels (fp32 state possible)
};

// defined in dg_tri.cu / dg_quad.cu / dg_tet.cu; nullptr if not compiled
Ops* ops_tri(int phys, int p);
Ops* ops_quad(int phys, int p);
Ops* ops_tet(int phys, int p);
Ops* ops_hyb(int phys, int p);

// Instantiation helper used by the per-kind translation units.
template <int K, int PH, int P>
struct Instance {
  using C = Cfg<K, PH, P>;
  using T = Tpe<C>;
  template <class S>
  static void launch_tpe(const View& v, S* U, S* R, const RK* rk, int64_t b, int64_t e, int grid,
                         cudaStream_t s, bool has_first, bool has_last) {
    const bool krk = rk && has_last;
    const RK r = rk ? *rk : RK{};
    if (krk && has_first)
      k_tpe_colored<C, PH, true, true, S><<<grid, T::THREADS, T::SMEM, s>>>(v, U, R, r, b, e);
    else if (krk)
      k_tpe_colored<C, PH, true, false, S><<<grid, T::THREADS, T::SMEM_SURF, s>>>(v, U, R, r, b, e);
    else if (has_first)
      k_tpe_colored<C, PH, false, true, S><<<grid, T::THREADS, T::SMEM, s>>>(v, U, R, r, b, e);
    else
      k_tpe_colored<C, PH, false, false, S><<<grid, T::THREADS, T::SMEM_SURF, s>>>(v, U, R, r, b, e);
  }
  static cudaError_t colored(const View& v, void* U, void* R, const RK* rk, int64_t b,
                             int64_t e, int grid, cudaStream_t s, bool has_first, bool has_last,
                             bool f32) {
    if constexpr (T::OK) {
      if (f32)
        launch_tpe<float>(v, static_cast<float*>(U), static_cast<float*>(R), rk, b, e, grid, s,
                          has_first, has_last);
      else
        launch_tpe<double>(v, static_cast<double*>(U), static_cast<double*>(R), rk, b, e, grid,
                           s, has_first, has_last);
    } else {
      if (f32) return cudaErrorNotSupported;
      double* Ud = static_cast<double*>(U);
      double* Rd = static_cast<double*>(R);
      if (rk)
        k_surface_colored<C, PH, true><<<grid, C::THREADS, C::SMEM, s>>>(v, Ud, Rd, *rk, b, e);
      else
        k_surface_colored<C, PH, false><<<grid, C::THREADS, C::SMEM, s>>>(v, Ud, Rd, RK{}, b, e);
    }
    return cudaGetLastError();
  }
  static cudaError_t volume(const View& v, const double* U, double* R, int grid,
                            cudaStream_t s) {
    if constexpr (T::OK)
      k_tpe_volume<C, PH><<<grid, T::THREADS, T::SMEM, s>>>(v, U, R);
    else
      k_volume<C, PH><<<grid, C::THREADS, C::VSMEM, s>>>(v, U, R);
    return cudaGetLastError();
  }
  static cudaError_t uncolored(const View& v, const double* U, double* out, bool atomic,
                               int grid, cudaStream_t s) {
    if constexpr (T::OK) {
      if (atomic)
        k_tpe_uncolored<C, PH, true><<<grid, T::THREADS, T::SMEM, s>>>(v, U, out);
      else
        k_tpe_uncolored<C, PH, false><<<grid, T::THREADS, T::SMEM, s>>>(v, U, out);
    } else {
      if (atomic)
        k_surface_uncolored<C, PH, true><<<grid, C::THREADS, C::SMEM, s>>>(v, U, out);
      else
        k_surface_uncolored<C, PH, false><<<grid, C::THREADS, C::SMEM, s>>>(v, U, out);
    }
    return cudaGetLastError();
  }
  static cudaError_t gather(const View& v, const double* buf, double* R, int cap,
                            cudaStream_t s) {
    const int64_t total = v.n_elements * C::NEQ * C::NP;
    int64_t g = (total + kThreads - 1) / kThreads;
    if (g > 148 * 16) g = 148 * 16;
    if (cap > 0 && g > cap) g = cap;
    if (g < 1) g = 1;
    k_gather<C><<<int(g), kThreads, 0, s>>>(v, buf, R);
    return cudaGetLastError();
  }
  static cudaError_t init(Ops* o) {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto fit = [&](const void* fn, int smem, int threads, int* grid) -> cudaError_t {
      cudaError_t e2 = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e2 != cudaSuccess) return e2;
      e2 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
      if (e2 != cudaSuccess) return e2;
      *grid = sms * (occ > 0 ? occ : 1);
      return cudaSuccess;
    };
    cudaError_t err;
    int g2 = 0;
    if constexpr (T::OK) {
      if ((err = fit((const void*)k_tpe_colored<C, PH, true, true>, T::SMEM, T::THREADS, &o->grid_var[3]))) return err;
      if ((err = fit((const void*)k_tpe_colored<C, PH, false, true>, T::SMEM, T::THREADS, &o->grid_var[1]))) return err;
      if ((err = fit((const void*)k_tpe_colored<C, PH, true, false>, T::SMEM_SURF, T::THREADS, &o->grid_var[2]))) return err;
      if ((err = fit((const void*)k_tpe_colored<C, PH, false, false>, T::SMEM_SURF, T::THREADS, &o->grid_var[0]))) return err;
      // the fp32-state instantiations share the grids (same launch bounds)
      for (const void* fn : {(const void*)k_tpe_colored<C, PH, true, true, float>,
                             (const void*)k_tpe_colored<C, PH, false, true, float>})
        if ((err = fit(fn, T::SMEM, T::THREADS, &g2))) return err;
      for (const void* fn : {(const void*)k_tpe_colored<C, PH, true, false, float>,
                             (const void*)k_tpe_colored<C, PH, false, false, float>})
        if ((err = fit(fn, T::SMEM_SURF, T::THREADS, &g2))) return err;
      o->grid_colored = o->grid_var[0];
      for (int k = 1; k < 4; ++k)
        if (o->grid_var[k] < o->grid_colored) o->grid_colored = o->grid_var[k];
      if ((err = fit((const void*)k_tpe_volume<C, PH>, T::SMEM, T::THREADS, &o->grid_volume))) return err;
      if ((err = fit((const void*)k_tpe_uncolored<C, PH, true>, T::SMEM, T::THREADS, &o->grid_uncolored))) return err;
      if ((err = fit((const void*)k_tpe_uncolored<C, PH, false>, T::SMEM, T::THREADS, &g2))) return err;
      if (g2 < o->grid_uncolored) o->grid_uncolored = g2;
    } else {
      if ((err = fit((const void*)k_surface_colored<C, PH, true>, C::SMEM, C::THREADS, &o->grid_colored))) return err;
      if ((err = fit((const void*)k_surface_colored<C, PH, false>, C::SMEM, C::THREADS, &g2))) return err;
      o->grid_var[2] = o->grid_var[3] = o->grid_colored;
      o->grid_var[0] = o->grid_var[1] = g2;
      if (g2 < o->grid_colored) o->grid_colored = g2;
      if ((err = fit((const void*)k_volume<C, PH>, C::VSMEM, C::THREADS, &o->grid_volume))) return err;
      if ((err = fit((const void*)k_surface_uncolored<C, PH, true>, C::SMEM, C::THREADS, &o->grid_uncolored))) return err;
      if ((err = fit((const void*)k_surface_uncolored<C, PH, false>, C::SMEM, C::THREADS, &g2))) return err;
      if (g2 < o->grid_uncolored) o->grid_uncolored = g2;
    }
    return cudaSuccess;
  }
  static cudaError_t stage_global(const double* tables, double* out, cudaStream_t s) {
    const int smem = C::S_TOTAL * 8;
    cudaError_t e = cudaFuncSetAttribute((const void*)k_stage_global<C>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k_stage_global<C><<<1, 256, smem, s>>>(tables, out);
    return cudaGetLastError();
  }
  static cudaError_t upload_const(const double* ptables_dev) {
    // the volume tables depend on (kind, degree) only: both physics share one
    return cudaMemcpyToSymbol(c_voltab<K, P>, ptables_dev + C::S_VPHI,
                              sizeof(double) * (C::S_SIZE - C::S_VPHI), 0,
                              cudaMemcpyDeviceToDevice);
  }
  static Ops* ops() {
    static Ops o{C::DIM, C::NEQ, C::NP, C::NQF, C::NQV, C::NCODES, C::T_SIZE,
                 T::OK ? T::THREADS : C::THREADS, T::OK ? T::SW : C::SPW,
                 0, 0, 0, {0, 0, 0, 0}, &colored, &volume, &uncolored, &gather, &init, C::S_TOTAL,
                 &stage_global, &upload_const, C::NPL, C::P1PROJ ? 1 : 0, T::OK ? 1 : 0};
    return &o;
  }
};

}  // namespace mcdg
