/*
 * meshchroma_b200 — C ABI of the B200 (sm_100a) colored surface-integral
 * hot path.  Plain pointers and sizes only; no torch types cross this
 * boundary.  Every function returns an int status (MC_OK == 0); on failure
 * mc_last_error() holds a message whose text matches the reference's
 * exception message where one exists.
 *
 * Reference interfaces replaced (reference = /root/reference/pkg/src/meshchroma):
 *   mc_color / mc_modified_greedy / mc_resolve_conflicts / mc_naive_greedy
 *       -> coloring.color :395-459, modified_greedy :351-362,
 *          resolve_conflicts :365-392, naive_greedy :462-488
 *   mc_layout_create / mc_layout_race_check
 *       -> sweeps.assert_race_free :89-105 (plus the color grouping that
 *          sweep_colored does per call at :144-149)
 *   mc_sweep_colored_i64[_host]      -> sweeps.sweep_colored :114-152
 *   mc_surface_buffer_i64            -> sweeps.surface_buffer :155-176
 *   mc_sweep_buffered_i64[_host]     -> sweeps.sweep_buffered :179-204
 *   mc_sweep_atomic_i64              -> (absent in the reference: SPEC.md:411;
 *                                        paper §1 "atomic operations")
 *   mc_assemble_create/_result       -> mesh.assemble :207-300 (surface ids,
 *                                        incidence, NonManifoldError :275-283)
 *   mc_amr_classify                  -> amr._materialize :221-245 + colors
 *                                        :158-164 (split-edge propagation)
 *   mc_dg_*                          -> Algorithm 1 / Eq. (2) of the paper
 *                                        (PAPER.md:29-33, 64-82); the
 *                                        reference implements only the
 *                                        integer stand-in (sweeps.py:1-24)
 *
 * Device pointers ("_dev") must be CUDA global memory on the current device;
 * "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).
 * "_host" entry points take host buffers and include the host<->device
 * copies (the end-to-end path a ctypes/cffi caller would use).
 */
#ifndef MESHCHROMA_B200_H_
#define MESHCHROMA_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to the reference's exception types) ---- */
#define MC_OK 0
#define MC_EINVAL 1        /* ValueError                                   */
#define MC_ECONFLICT 2     /* WriteConflictError (errors.py:48-49)         */
#define MC_ESWAPBUDGET 3   /* SwapBudgetExceededError (errors.py:24-25)    */
#define MC_ERESTARTS 4     /* RestartsExhaustedError (errors.py:28-29)     */
#define MC_EAUDIT 5        /* AssertionError from audit mode               */
#define MC_EINTERNAL 6     /* AssertionError (broken invariant)            */
#define MC_ECUDA 7         /* CUDA runtime failure                         */
#define MC_ENOMEM 8        /* allocation failure                           */
#define MC_EUNSUPPORTED 9  /* configuration without a compiled kernel      */
#define MC_ENONMANIFOLD 10 /* NonManifoldError (errors.py; mesh.py:283-290) */

const char* mc_last_error(void);
/* 1000*major + 10*minor of the library; lets bindings check the ABI. */
int mc_abi_version(void);
/* Number of CUDA devices visible (0 on a CPU-only host; never fails). */
int mc_device_count(void);

/* ------------------------------------------------------------------ */
/* Coloring (host C++, bit-exact with CPython random.Random streams)   */
/* ------------------------------------------------------------------ */
typedef struct mc_coloring_stats {
  int64_t greedy_conflicts;
  int64_t resolutions;
  int64_t swaps;
  int64_t loop_breaks;
  int64_t no_swap_breaks;
  int64_t forced_reswaps;
  int64_t restarts;
  double greedy_seconds;
  double resolve_seconds;
  double total_seconds;
} mc_coloring_stats;

/* surf_elems: (ns, 2) int64 row-major, right = -1 on the boundary.
 * elem_surfs: (ne, 4) int64 row-major, -1 padded.
 * chain_budget < 0 selects the reference default 10 * ns; the total budget
 * is 5 * chain_budget (coloring.py:410-412, 429-431). */
int mc_color(int64_t n_surfaces, int64_t n_elements, const int64_t* surf_elems,
             const int64_t* elem_surfs, int n_colors, int64_t seed,
             int64_t chain_budget, int max_restarts, int audit,
             int32_t* colors_out, mc_coloring_stats* stats);
int mc_modified_greedy(int64_t n_surfaces, int64_t n_elements,
                       const int64_t* surf_elems, int n_colors, int64_t seed,
                       int32_t* colors_out, int64_t* n_conflicts);
int mc_resolve_conflicts(int64_t n_surfaces, int64_t n_elements,
                         const int64_t* surf_elems, const int64_t* elem_surfs,
                         int n_colors, int64_t seed, int64_t chain_budget,
                         int audit, int32_t* colors_inout,
                         mc_coloring_stats* stats);
int mc_naive_greedy(int64_t n_surfaces, int64_t n_elements,
                    const int64_t* surf_elems, int32_t* colors_out,
                    int32_t* n_colors_out);

/* ------------------------------------------------------------------ */
/* Color-major device layout + integer sweeps (Algorithm 1, int64)     */
/* ------------------------------------------------------------------ */
typedef struct mc_layout mc_layout;

/* Groups surfaces by color (stable: ascending surface id inside a color,
 * like sweeps.py:145) and uploads incidence to the device.  colors must be
 * >= 1 (complete); colors > n_colors are never swept, as in the reference
 * loop bound (sweeps.py:144). */
int mc_layout_create(int64_t n_surfaces, int64_t n_elements,
                     const int64_t* surf_elems, const int64_t* elem_surfs,
                     const int32_t* colors, int n_colors, mc_layout** out);
int mc_layout_destroy(mc_layout* layout);
/* Number of surfaces in color c (1-based); -1 on a bad color. */
int64_t mc_layout_color_size(const mc_layout* layout, int color);

/* Device race certificate: for the first color (ascending) in which some
 * element is written twice, reports the smallest such element id and its
 * write count and returns MC_ECONFLICT with the reference message
 * "color c writes element e k times" (sweeps.py:102-105). */
int mc_layout_race_check(mc_layout* layout, void* stream);

/* totals_dev (ne) is overwritten.  One kernel launch per color, stream
 * order is the inter-color barrier. */
int mc_sweep_colored_i64(mc_layout* layout, const int64_t* payload_dev,
                         int64_t* totals_dev, void* stream);
int mc_surface_buffer_i64(mc_layout* layout, const int64_t* payload_dev,
                          int64_t* buffer_dev /* 2*ns */, void* stream);
int mc_sweep_buffered_i64(mc_layout* layout, const int64_t* payload_dev,
                          int64_t* buffer_dev /* 2*ns scratch */,
                          int64_t* totals_dev, void* stream);
int mc_sweep_atomic_i64(mc_layout* layout, const int64_t* payload_dev,
                        int64_t* totals_dev, void* stream);
/* Host-buffer variants: H2D payload, sweep, D2H totals, synchronize.
 * strategy: 0 colored, 1 buffered, 2 atomic. */
int mc_sweep_i64_host(mc_layout* layout, int strategy,
                      const int64_t* payload_host, int64_t* totals_host);
/* Splitmix64 payload on the device (sweeps.py:55-62). */
int mc_default_payload_dev(int64_t n, int64_t seed, int64_t* out_dev,
                           void* stream);

/* ------------------------------------------------------------------ */
/* DG surface integral (Eq. (2) of the paper) in fp64                  */
/* ------------------------------------------------------------------ */
#define MC_KIND_TRI 0
#define MC_KIND_QUAD 1
#define MC_KIND_TET 2
/* conforming triangle + quadrilateral mix (2D); element blocks have the
 * quad basis size, triangles use its first (p+1)(p+2)/2 modes per equation
 * (the rest stay zero); face codes 0-23 quad sides, 24-41 triangle sides;
 * volume tables: the quad rule's rows, then the triangle rule's */
#define MC_KIND_HYBRID 3
#define MC_PHYS_ADVECTION 0
#define MC_PHYS_EULER 1

#define MC_DG_COLORED 0
#define MC_DG_BUFFERED 1
#define MC_DG_ATOMIC 2

/* per-surface code word */
#define MC_SIDE_CODE_BITS 6
#define MC_FLAG_L_FIRST (1u << 12)
#define MC_FLAG_L_LAST (1u << 13)
#define MC_FLAG_R_FIRST (1u << 14)
#define MC_FLAG_R_LAST (1u << 15)
#define MC_FLAG_R_GHOST (1u << 16)
/* sides swapped w.r.t. the canonical (single-domain) orientation by the
 * partitioner: the flux is evaluated in canonical orientation so owned
 * residuals stay bit-identical to the single-domain run */
#define MC_FLAG_FLIPPED (1u << 17)

typedef struct mc_dg_desc {
  int kind;        /* MC_KIND_* */
  int physics;     /* MC_PHYS_* */
  int degree;      /* polynomial degree p */
  int n_colors;
  int64_t n_elements;      /* owned elements (written)            */
  int64_t n_ghosts;        /* read-only ghost elements after them */
  int64_t n_surfaces;      /* surfaces in the color-major list    */
  const int64_t* group_bounds;     /* n_colors+1 prefix sums (host)     */
  const int32_t* surf_left;        /* ns                                */
  const int32_t* surf_right;       /* ns, -1 = physical boundary        */
  const uint32_t* surf_code;       /* ns, side codes + flags            */
  const double* surf_geom;         /* ns x (dim+2): n_0..n_{d-1}, sL, sR */
  const double* elem_jinv;         /* (ne+ng) x dim x dim, dxi_r/dx_d   */
  const int64_t* elem_slot_ptr;    /* ne+1 CSR offsets (buffered gather) */
  const int32_t* elem_slots;       /* buffer slots 2*s+side per element,
                                      local side order                    */
  /* reference-element tables (host), see dg/tables.py */
  int n_face_codes, n_face_q, n_vol_q, n_basis;
  const double* face_phi;  /* n_face_codes x n_face_q x n_basis */
  const double* face_w;    /* n_face_q                            */
  const double* vol_phi;   /* n_vol_q x n_basis                   */
  const double* vol_dphi;  /* dim x n_vol_q x n_basis             */
  const double* vol_w;     /* n_vol_q                             */
  /* physics */
  double gamma;
  double velocity[3];
  double farfield[5];
  /* state storage: 0 = fp64 element blocks; 1 = fp32 blocks (all arithmetic
   * stays fp64; colored strategy and steppers only; the north star's
   * 1e-5 tolerance).  Every U / U0 / R / work / send-buffer pointer of an
   * fp32 operator points to floats, strides count floats. */
  int state_f32;
  /* MC_KIND_HYBRID: per element (ne+ng) 0 = triangle, 1 = quad; else NULL */
  const uint8_t* elem_kind;
} mc_dg_desc;

typedef struct mc_dg mc_dg;

int mc_dg_create(const mc_dg_desc* desc, mc_dg** out);
int mc_dg_destroy(mc_dg* dg);
/* doubles between consecutive element blocks (block padded to 32 B) */
int64_t mc_dg_block_stride(const mc_dg* dg);
int64_t mc_dg_buffer_bytes(const mc_dg* dg); /* buffered-variant scratch */
/* Upper bound on the blocks of every persistent-grid launch (0 = the
 * occupancy-sized default).  A small cap makes every warp loop over many
 * surface tiles even on a small mesh (the loop-carried path production
 * runs), which is what the parity tests use it for. */
int mc_dg_set_grid_cap(mc_dg* dg, int max_blocks);

/* R := RHS(U) on owned elements.  Colored: volume fused into each
 * element's first color pass, surfaces one launch per color, no atomics,
 * no buffer.  Buffered/atomic: the paper's comparison strategies. */
int mc_dg_rhs(mc_dg* dg, const double* U_dev, double* R_dev, int strategy,
              void* stream);
/* One fused SSP-RK stage: U <- a*U0 + b*(U + dt*RHS(U)), in place,
 * volume fused into first-touch passes, update fused into last-touch
 * passes.  R_scratch_dev holds partial sums between color passes. */
int mc_dg_rk_stage(mc_dg* dg, double* U_dev, const double* U0_dev,
                   double* R_scratch_dev, double a, double b, double dt,
                   void* stream);
/* One color launch of the colored strategy (what mc_dg_rhs / rk_stage /
 * ssprk3 issue n_colors times); rk_mode 0 = residual only, 1 = RK stage
 * update in last-touch sides, 2 = as 1 and save U0 := U first.  Exposed so
 * callers can time or interleave individual color launches. */
int mc_dg_color_pass(mc_dg* dg, int color, double* U_dev, double* U0_dev,
                     double* R_dev, int rk_mode, double a, double b, double dt,
                     void* stream);
/* As mc_dg_color_pass over surfaces [begin, end) of the color's list
 * (relative to the color's first surface).  A partitioned layout puts the
 * surfaces that touch ghost elements last in every color, so the interior
 * part of the first color can run while the ghost exchange is in flight. */
int mc_dg_color_range_pass(mc_dg* dg, int color, int64_t begin, int64_t end,
                           double* U_dev, double* U0_dev, double* R_dev, int rk_mode,
                           double a, double b, double dt, void* stream);
/* Partitioned runs: slot[e] (n_elements entries, -1 = none) names the row of
 * the caller's ghost-exchange send buffer (n_slots blocks of `stride`
 * doubles, device memory) that owned element e is sent from.  Every
 * last-touch pass of an RK stage then also stores e's updated block there,
 * so the next stage's exchange posts the buffer without a gather.  slot =
 * NULL turns it off. */
int mc_dg_set_send_rows(mc_dg* dg, const int32_t* slot_host, double* send_buf_dev,
                        int64_t n_slots);
/* Peer-push ghost exchange (partitioned runs on one NVLink/NVSwitch node):
 * dst[ptr[e] .. ptr[e+1]) are byte addresses, valid in this process (peer
 * memory mapped by the caller, e.g. symmetric memory), of the rows that
 * owned element e's block must land in on the peers; every last-touch pass
 * of an RK stage stores e's updated block there (+ the push parity's row
 * shift) as it writes U — the exchange is fused into the kernel, no send
 * buffer, no copy engine.  ptr = NULL turns it off.  Register kernels only. */
int mc_dg_set_push_rows(mc_dg* dg, const int64_t* ptr_host, const uint64_t* dst_host,
                        int64_t nnz);
/* Double-buffered ghost rows for the peer push: ghost g (id ne + g in the
 * surface list) lives at rows ne + 2g (parity 0) and ne + 2g + 1 (parity 1)
 * of U; launches read read_parity (-1: the plain layout, ghost g at row
 * ne + g) and push into the peers' push_parity rows.  A stage reads the
 * parity its peers pushed in the previous stage and pushes the other one,
 * so a peer still reading this stage's ghosts is never overwritten. */
int mc_dg_set_ghost_parity(mc_dg* dg, int read_parity, int push_parity);
/* n_steps SSP-RK3 steps; work_dev = 2 blocks arrays (U0, R scratch). */
int mc_dg_ssprk3(mc_dg* dg, double* U_dev, double* work_dev, double dt,
                 int n_steps, void* stream);
/* End-to-end: copy U from host, n_steps SSP-RK3 steps, copy back (U_host
 * in the internal layout). */
int mc_dg_ssprk3_host(mc_dg* dg, double* U_host, double dt, int n_steps);

/* Caller (user) element order — what the reference-facing API takes:
 * arrays of n_user_rows x (N_eq * N_p) doubles, one unpadded row per element
 * in the caller's numbering.  src[r] (n_elements entries) is the user row
 * of internal owned row r (the inverse of reorder.build_plan's
 * element_perm for a single domain; the owned global ids on a partition). */
int mc_dg_set_user_rows(mc_dg* dg, const int64_t* src_host, int64_t n_user_rows);
/* Device permutations between the two layouts (internal padding zeroed). */
int mc_dg_user_to_internal(mc_dg* dg, const double* user_dev, double* U_dev, void* stream);
int mc_dg_internal_to_user(mc_dg* dg, const double* U_dev, double* user_dev, void* stream);
/* End-to-end in the user layout (DGOperator.ssprk3 / .rhs): H2D of the
 * caller's array, device permutation, the colored steps (or one RHS with the
 * given strategy), permutation back, D2H.  Single-domain operators only. */
int mc_dg_ssprk3_user_host(mc_dg* dg, double* U_user_host, double dt, int n_steps);
int mc_dg_rhs_user_host(mc_dg* dg, const double* U_user_host, double* R_user_host,
                        int strategy);

/* ------------------------------------------------------------------ */
/* Surface extraction (mesh.assemble, reference mesh.py:207-300)       */
/* ------------------------------------------------------------------ */
/* Side slots sorted by packed vertex key on the GPU (CUB radix sort),
 * surfaces numbered by first encounter in element-major slot order, left =
 * smaller element id.  Inputs are HOST arrays already validated by the
 * caller (kind codes 0..2, vertex ids in range, no repeated vertices).
 * Returns MC_ENONMANIFOLD (handle still valid: fetch surf_count to report)
 * when a surface has more than two elements, MC_EUNSUPPORTED when the
 * packed key does not fit 64 bits. */
typedef struct mc_assembly mc_assembly;
int mc_assemble_create(int64_t n_elements, int64_t n_vertices, const int8_t* kind_codes,
                       const int64_t* elem_verts /* n_elements x 4 */, int width,
                       mc_assembly** out, int64_t* n_surfaces);
/* host outputs (any may be NULL): surf_verts n_surfaces x width (sorted
 * tuples), surf_elems n_surfaces x 2, elem_surfs n_elements x 4 (-1 pad),
 * surf_count n_surfaces (elements per surface) */
int mc_assemble_result(mc_assembly* a, int64_t* surf_verts, int64_t* surf_elems,
                       int64_t* elem_surfs, int32_t* surf_count);
int mc_assemble_destroy(mc_assembly* a);

/* ------------------------------------------------------------------ */
/* AMR split-edge color propagation (amr._materialize classification,  */
/* reference amr.py:221-245 + :158-164)                                */
/* ------------------------------------------------------------------ */
/* Host arrays in and out.  fine_surf_verts: n_fine_surfaces x 2 sorted
 * (midpoint vertex ids are n_base_vertices + index into split); split: the
 * base edges that were split, ascending.  Outputs per fine surface: origin
 * (0 whole, 1 half, 2 interior), related base edge, half index (1/2, else
 * 0) and the 6-palette color.  MC_EINTERNAL (AssertionError) when a fine
 * edge has no base counterpart. */
int mc_amr_classify(int64_t n_fine_surfaces, const int64_t* fine_surf_verts,
                    int64_t n_base_vertices, int64_t n_split, const int64_t* split,
                    int64_t n_base_surfaces, const int64_t* base_surf_verts,
                    const int32_t* base_colors, int8_t* surf_origin, int64_t* base_surface,
                    int8_t* half_index, int32_t* colors);

#ifdef __cplusplus
}
#endif
#endif /* MESHCHROMA_B200_H_ */
