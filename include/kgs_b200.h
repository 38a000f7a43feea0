/*
 * kgs_b200.h -- C ABI of the B200-native checkerboard DP-AVF2 stepper for the
 * Klein-Gordon-Schrodinger system (arXiv 2502.09537).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (pure Python + numba, /root/reference/pkg/src/dpavf) drives the sweep
 * through two operator layers that cannot survive on a device unchanged:
 *
 *   executor.run(schedule, lane_fn)          dpavf/executor.py:39-40, 60-71
 *   kernels.sweep_base / sweep_adjoint(P,Q,U,V,nbrs,order, 11 coeffs)
 *                                            dpavf/kernels.py:23-54, 57-94
 *
 * Both are gather "lanes" over host index arrays (an (M,2d) int64 neighbour
 * table plus an int64 order), so the replacement sits one level up, at the
 * colour granularity used by step_base / step_adjoint / step_dpavf2 /
 * integrate (dpavf/integrator.py:107-182) and discrete_energy / mass /
 * FieldState.is_finite (dpavf/grid.py:101-103, 166-187).  Each entry point
 * below names the reference function it replaces.
 *
 * Conventions
 *   - Host field arrays are float64, length (planes owned) * N^(d-1), in the
 *     reference linearisation i = x*N^(d-1) + y*N^(d-2) + z (first axis
 *     slowest, dpavf/grid.py:4-7).  Copy semantics: the caller keeps
 *     ownership of host memory; the context owns device memory.
 *   - Colour: 1 = red (index-sum parity 1, swept first by the base sweep),
 *     0 = black (dpavf/ordering.py:114-136, 139-149).
 *   - Kind:   0 = base sweep (kernels.sweep_base), 1 = adjoint sweep
 *     (kernels.sweep_adjoint).
 *   - Every call is synchronous at return (results visible to the host).
 *   - Return 0 on success or a negative KGS_E* code; kgs_last_error() holds
 *     a message.  A context is used by one host thread at a time.
 */
#ifndef KGS_B200_H
#define KGS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KGS_OK 0
#define KGS_EINVAL (-1)     /* bad argument: odd N, d not in {1,2,3}, bad split */
#define KGS_ECUDA (-2)      /* CUDA runtime error (message in kgs_last_error) */
#define KGS_ENCCL (-3)      /* NCCL error or NCCL not loadable */
#define KGS_ENONFINITE (-4) /* non-finite field values detected */
#define KGS_ENOMEM (-5)     /* device allocation failed */

#define KGS_NTERMS 8        /* energy/mass term sums, see kgs_energy_terms */

typedef struct kgs_ctx kgs_ctx;

/* The 11 kernel scalars in StepCoefficients.kernel_args() order
 * (dpavf/integrator.py:42-45): alpha, beta, gcoef, c_uv, uv_nbr, gU,
 * half_tau (= coeffs.tau / 2), i00, i01, i10, i11.  Computed on the host
 * exactly as precompute_coefficients (dpavf/integrator.py:48-64). */
typedef struct kgs_coeffs {
  double alpha, beta, gcoef, c_uv, uv_nbr, gU, half_tau, i00, i01, i10, i11;
} kgs_coeffs;

/* ---- context lifetime ------------------------------------------------- */

/* Single-process context over the whole periodic grid GridSpec(d, a, b, N)
 * (dpavf/grid.py:16-64).  The grid is split into `nslabs` slabs of N/nslabs
 * planes along axis 0; slab s lives on device dev_ids[s] (several slabs may
 * share one device: "virtual slabs", used to test decomposition invariance
 * on one GPU).  nslabs == 1 is the ordinary single-GPU case.
 * KGS_EINVAL: d not in {1,2,3}, N < 2, N odd (checkerboard needs even N,
 * dpavf/ordering.py:120-122), nslabs < 1, N % nslabs != 0, N/nslabs < 2 when
 * nslabs > 1, or nslabs > 1 with d == 1. */
int kgs_create(int d, int64_t N, double a, double b, int nslabs,
               const int* dev_ids, kgs_ctx** out);

/* One rank of a multi-process run (one process per GPU, torchrun): this
 * context owns slab `rank` of `nranks` on `device`; face halos travel over
 * NCCL send/recv to ranks rank-1 / rank+1 (periodic).  `nccl_id` is the
 * 128-byte ncclUniqueId produced by kgs_nccl_unique_id on rank 0 and
 * broadcast by the caller.  nranks == 1 needs no NCCL (nccl_id may be NULL).
 * Test hook: nranks == 1 with a non-NULL nccl_id and KGS_SELF_EXCHANGE=1 in
 * the environment makes the single slab exchange its faces with itself over
 * NCCL instead of wrapping in the kernel -- the multi-rank code path (ghost
 * planes, interior/boundary split, send/recv on the comm stream, event
 * waits) run on one GPU. */
int kgs_create_dist(int d, int64_t N, double a, double b, int rank, int nranks,
                    int device, const void* nccl_id, kgs_ctx** out);

/* Fill 128 bytes with a fresh ncclUniqueId (rank 0 only). */
int kgs_nccl_unique_id(void* out128);

int kgs_destroy(kgs_ctx* ctx);

/* Planes [*x0, *x0 + *nx) along axis 0 owned by this context (whole grid for
 * kgs_create; one slab for kgs_create_dist); *points = nx * N^(d-1). */
int kgs_local_range(kgs_ctx* ctx, int64_t* x0, int64_t* nx, int64_t* points);

/* ---- state transfer (FieldState P, Q, U, V; dpavf/grid.py:82-103) ------ */

/* Host -> device copy of the owned planes (natural layout); the context
 * re-lays the fields out on the device (colour-split planes). */
int kgs_upload(kgs_ctx* ctx, const double* P, const double* Q,
               const double* U, const double* V);
/* Device -> host copy of the owned planes (natural layout). */
int kgs_download(kgs_ctx* ctx, double* P, double* Q, double* U, double* V);

/* Plane-range transfers of ONE field (0 P, 1 Q, 2 U, 3 V): planes
 * [x_begin, x_begin + nplanes) (global axis-0 indices inside this context's
 * range), natural layout, nplanes * N^(d-1) doubles.  Used to stream KGS1
 * snapshots (dpavf/snapshot.py:30-64) without a full host copy. */
int kgs_upload_planes(kgs_ctx* ctx, int field, int64_t x_begin, int64_t nplanes,
                      const double* src);
int kgs_download_planes(kgs_ctx* ctx, int field, int64_t x_begin, int64_t nplanes,
                        double* dst);

/* ---- the hot path ------------------------------------------------------ */

/* One colour half of one sweep, in place: the device equivalent of
 * executor.run over one phase of checkerboard_schedule with lane_fn =
 * kernels.sweep_base (kind 0) or kernels.sweep_adjoint (kind 1).
 * step_base = sweep(red, base) then sweep(black, base); step_adjoint =
 * sweep(black, adjoint) then sweep(red, adjoint)
 * (dpavf/integrator.py:107-121, dpavf/ordering.py:139-149). */
int kgs_sweep(kgs_ctx* ctx, int colour, int kind, const kgs_coeffs* c);

/* `nsteps` DP-AVF2 steps (step_dpavf2 = base then adjoint at tau/2,
 * dpavf/integrator.py:124-129) -- the loop body of integrate
 * (dpavf/integrator.py:167-179) -- with fused colour passes.  The steps are
 * numbered n = step_offset + 1 .. step_offset + nsteps (global step numbers
 * of an integrate run split into several calls).
 * Every step is checked for non-finite values (integrate:169-171); if any
 * appear, *first_bad_step receives the first bad global step number and the
 * call returns KGS_ENONFINITE after finishing the launched work; otherwise
 * *first_bad_step = 0.
 * When record_stride > 0, the energy/mass term sums (see kgs_energy_terms)
 * of the state after every step n with n % record_stride == 0 are written,
 * in step order, to terms_out[r * KGS_NTERMS + q], r = 0, 1, ...
 * terms_out may be NULL when no step is recorded.
 * flags & KGS_STEP_DEFER_TAIL: the red adjoint half of the last step (unless
 * that step is recorded) is left pending in the context and fused into the
 * next call's first pass when the coefficients are equal -- 2 instead of 3
 * passes per step for step-at-a-time callers.  Results are bitwise the same;
 * every other entry point applies a pending adjoint first, and the last
 * step is then not checked for finiteness (step_dpavf2 does not check). */
#define KGS_STEP_DEFER_TAIL 1
/* flags & KGS_STEP_BACKUP: first copy the state at step_offset (a pending
 * tail applied) into the context's second buffer set (allocated on first
 * use; skipped when it does not fit), so that after KGS_ENONFINITE the
 * caller can kgs_restore_backup() and replay exactly to the first bad step
 * -- integrate()'s contract that the state is left after that step
 * (integrator.py:169-171).  Costs one device copy of the state. */
#define KGS_STEP_BACKUP 8
int kgs_step_dpavf2(kgs_ctx* ctx, const kgs_coeffs* half, int64_t nsteps,
                    int64_t step_offset, int64_t record_stride,
                    double* terms_out, int64_t* first_bad_step, int flags);

/* A whole integrate() call on a HOST state (dpavf/integrator.py:147-182):
 * upload P, Q, U, V, record the initial energy terms (terms0[8]), run
 * `nsteps` DP-AVF2 steps recording every `record_stride` steps into
 * terms_out[nrec][8] as kgs_step_dpavf2 does, and write the final state back
 * into the same host arrays (this context's planes, kgs_upload's convention).
 * The upload, the colour passes and the download are overlapped as a
 * pipeline (chunks of planes arrive around plane 0; every pass advances one
 * plane behind its predecessor; finished chunks are copied back while later
 * ones still compute), on every slab side by side with the faces exchanged
 * between the passes (kgs_pipeline_plan, split = 1); pageable arrays are
 * staged through page-locked slots by helper threads.  The ranks of a
 * torchrun job (kgs_create_dist) agree through NCCL on running the pipeline
 * and on the first bad step -- every rank must make this call; terms0 /
 * terms_out are then this rank's sums.  Without memory for the pipeline (or
 * knob "pipeline" = 0) the same result comes from upload + kgs_step_dpavf2
 * + download.  Fields are bitwise the same either way.  KGS_ENONFINITE: the
 * host arrays hold the state after step *first_bad_step (replayed exactly),
 * like the reference's integrate.  Knobs: "pipeline" (1/0),
 * "pipeline_planes", "stage_pageable" (1/0). */
int kgs_integrate_host(kgs_ctx* ctx, double* P, double* Q, double* U, double* V,
                       const kgs_coeffs* half, int64_t nsteps, int64_t step_offset,
                       int64_t record_stride, double* terms0, double* terms_out,
                       int64_t* first_bad_step, int flags);

/* The schedule kgs_integrate_host executes for N (local) planes, chunks of C
 * planes and nsteps steps, as events (kind, index, a, b) written to
 * out[4 * i ..] (at most `cap` events): kind 0 = chunk `index` (planes
 * [a, b)) arrived, 1 = pass `index` over planes [a, b) (passes: 0 black
 * energy terms, 1 red energy terms, 2 head, then K3/K4 per step), 2 = block
 * `index` (planes [a, b)) final and copied back, 3 (split = 1: several slabs
 * or ranks, every one running this plan on its own planes) = exchange the
 * faces pass `index` wrote (-1: both colours of the arrived state).  Pure
 * host logic (no device); returns the number of events, -1 on bad
 * arguments. */
int64_t kgs_pipeline_plan(int64_t N, int64_t C, int64_t nsteps, int split, int64_t* out,
                          int64_t cap);

/* The pass program kgs_step_dpavf2 executes on every slab / rank of `nx`
 * local planes (split = 1: several slabs or ranks, faces exchanged; 0: one
 * slab, x wraps in the kernel) -- the same list, from the same function.
 * Rows of 9 int64 (kind, col, op1, op2, diag, check, step, xa, xb) written to
 * out[9 * i ..] (at most `cap` rows):
 *   1 LAUNCH      colour `col` pass over local planes [xa, xb): op1 then op2
 *                 (0 none, 1 base, 2 adjoint), energy terms (diag) after the
 *                 adjoint, finiteness check (check) tagged with `step`
 *   2 WAIT_XCH    wait until the pending halo exchange has landed
 *   3 XCH         start the exchange of colour `col` faces: send P, Q, U of
 *                 plane 0 to rank-1 and of plane nx-1 to rank+1, receive
 *                 into ghost planes nx (from rank+1) and -1 (from rank-1)
 *   4 RECORD      reduce the energy partials into record slot `step`
 *   5 DEFER       the last red adjoint is left pending
 *   6 PASS_BEGIN / 7 PASS_END   bracket one colour pass (xa = 1: timed)
 * flags: KGS_STEP_DEFER_TAIL, KGS_PROGRAM_HEAD_FUSED (the previous call left
 * its red adjoint pending with the same coefficients).  Mirrors
 * integrator.py:167-179 (the DP-AVF2 loop) over dpavf/executor.py:60-71
 * (phases separated by barriers; here by exchanges and stream events).
 * Pure host logic; returns the number of rows, -1 on bad arguments. */
#define KGS_PROGRAM_HEAD_FUSED 2
int64_t kgs_step_program(int64_t nx, int split, int64_t nsteps, int64_t step_offset,
                         int64_t record_stride, int flags, int64_t* out, int64_t cap);

/* ---- diagnostics (dpavf/grid.py:152-187) ------------------------------- */

/* Unscaled sums over this context's points, deterministic for a given
 * decomposition (fixed-order warp/block/grid tree):
 *   t[0] = sum (P(i+e_ax) - P(i))^2 over all forward edges   (_grad_sq_sum*h^2)
 *   t[1] = same for Q, t[2] = same for U
 *   t[3] = V.V, t[4] = U.U, t[5] = (P^2+Q^2).U, t[6] = P.P, t[7] = Q.Q
 * discrete_energy = h^d * (0.5*(k1*(t0+t1)/h^2 + k2*t2/h^2 + t3 + mu^2*t4)
 *                          - gamma*t5),  mass = h^d * (t6 + t7). */
/* Restore the state saved by the last kgs_step_dpavf2(..., KGS_STEP_BACKUP)
 * call (KGS_EINVAL if there is none, or the state changed since through
 * another entry point). */
int kgs_restore_backup(kgs_ctx* ctx);

int kgs_energy_terms(kgs_ctx* ctx, double* terms_out);

/* discrete_energy(state, params, grid) and mass(state, grid) for the
 * resident state (single-process contexts; dist contexts return the local
 * slab's contribution). */
int kgs_energy_mass(kgs_ctx* ctx, double kappa1, double kappa2, double mu,
                    double gamma, double* E, double* mass);

/* FieldState.is_finite (dpavf/grid.py:101-103) for the resident state. */
int kgs_all_finite(kgs_ctx* ctx, int* ok);

/* Message for the last failing call on ctx (or the last global failure when
 * ctx is NULL). Never NULL. */
const char* kgs_last_error(kgs_ctx* ctx);

/* ---- benchmarking / introspection ------------------------------------- */

/* Number of kernel launches issued by this context since creation. */
int64_t kgs_launch_count(kgs_ctx* ctx);

/* Device time in milliseconds of the most recent kgs_step_dpavf2 call,
 * measured with CUDA events on the context's stream(s) (max over slabs). */
double kgs_last_step_ms(kgs_ctx* ctx);

/* Tile/grid tuning of the colour passes (defaults 4, 64, 0, 0, 0): rows
 * per 256-thread tile of the simple kernel (power of two), band height in
 * rows for its band-major tile order (<= 0: plane-major), a cap on resident
 * blocks per SM (0: occupancy maximum), planes per work unit of the 3-D
 * marching kernel (0: automatic, < 0: never use the marching kernel), and
 * the marching kernel's variant (0: 4x64 rows x slots, one point per
 * thread; 1: 8x64, one point per thread; 4, the default: 8x64, two rows per
 * thread at 2 CTAs/SM; the other shapes 2, 3, 5..12 and the clustered /
 * producer-warp variants 13..15 exist only in experimental builds; < 0:
 * keep).
 * Results do not depend on these (bitwise). */
int kgs_set_tuning(kgs_ctx* ctx, int rows_per_tile, int band_rows, int blocks_per_sm,
                   int march_planes, int march_variant);

/* Named tuning knob (results never depend on it): "march_variant",
 * "march_planes", "march_wave_sync" (1, the default: a software grid
 * barrier after every wave of work units of the marching kernel, so
 * neighbouring columns march together and their shared halo rows / columns
 * are re-read from L2 -- a bounded-spin performance heuristic, off for
 * several slabs per GPU and inside kgs_integrate_host; 0: free-running),
 * "march_sync" (planes between cluster barriers of the
 * clustered variants), "blocks_per_sm", "march_sms" (SMs the march grid
 * spans; 0 = all), "record_form" (3-D record passes, the red colour's
 * gradient terms: 2 = sums of squares of the neighbour values the update
 * loads, completed with the new value -- the default, fastest; 1 = from the
 * differences to the pre-update value, free of cancellation for fields with
 * a large offset; records only, fields identical), "fused_step" (1: one fused march
 * per DP-AVF2 step -- K3 and K4 with ping-pong buffer sets, allocated on
 * first use; 3-D, rows % 16 == 0, slots % 32 == 0 -- bitwise equal but
 * currently slower; 0, the default: two colour passes), "fused_planes"
 * (fused step: K4 planes per work unit, default 128), "fused_debug"
 * (timing experiments only, CORRUPTS results: 1 no ring K3, 2 no K4
 * arithmetic, 4 no K3 arithmetic), "resident" (1, the default: a grid
 * whose state fits in one CTA's shared memory -- 32 B per point <= 200 KiB
 * -- runs a whole kgs_step_dpavf2 call in one launch; 0: per-pass
 * launches), "mirror_halo" (1, the default: single-process slabs store
 * their faces from the boundary launches straight into the neighbours'
 * ghost planes; 0: peer copies after each pass), "tma_store" (marching
 * kernel's own-tile write: 0 per-thread stores, 1 one TMA bulk store, 2,
 * the default, bulk store with an L2 evict-first hint), "pipeline" (1, the
 * default: kgs_integrate_host overlaps upload, passes and download on one
 * slab; 0: in sequence), "pipeline_planes" (its chunk in planes; 0, the
 * default: 16 for page-locked arrays when the per-record partials fit,
 * else 32), "pdl" (1, the default: the colour passes are launched as
 * programmatic dependents of the previous kernel on the stream, so their
 * launch and set-up overlap its drain; 0: plain stream order; record
 * reductions run on a per-slab record stream either way).
 * KGS_EINVAL for unknown names. */
int kgs_set_param(kgs_ctx* ctx, const char* name, int value);

/* L2 sector promotion of the marching kernel's TMA boxes (0 none, 1 64 B,
 * 2 128 B, 3 256 B) for the other-colour halo box and the own tile box;
 * default 0, 0.  Results do not depend on it. */
int kgs_set_promotion(kgs_ctx* ctx, int halo, int tile);

/* Benchmarking only (CORRUPTS the resident state): average device time of
 * `reps` black fused passes of the marching kernel in a debug mode:
 * 0 = normal, 1 = no arithmetic (data movement only), 2 or 3 = no stores.
 * Used to measure the pass's memory ceiling. */
int kgs_debug_pass(kgs_ctx* ctx, int mode, int reps, double* ms_out);

/* Device self-test: the shared-reciprocal division used by the kernels
 * against the IEEE `/` on n pseudo-random operand pairs; *mismatches
 * counts bitwise differences (expected 0). */
int kgs_selftest_division(int device, int64_t n, uint64_t seed, int64_t* mismatches);

/* Per-launch timing of the fused launches inside kgs_step_dpavf2 (colour
 * passes K3 / K4, or one-sweep steps): when enabled, a CUDA event pair
 * brackets each such launch on its stream.  kgs_pass_stats returns the
 * number of timed launches and their summed device time (ms) since the
 * last kgs_pass_timing call, and the points each launch updated twice
 * (one colour for a pass, the whole grid for a sweep). */
int kgs_pass_timing(kgs_ctx* ctx, int enable);
int kgs_pass_stats(kgs_ctx* ctx, int64_t* launches, double* total_ms,
                   int64_t* points_per_launch);

/* Fill the resident state on the device from a named initial condition
 * (0 = ellipsoids3d, 1 = fourpeak2d, 2 = gaussian2d, 3 = soliton1d) without
 * a host round trip; used for >= 512^3 benchmark inputs.  Values agree with
 * the numpy presets to libm rounding, not bitwise. */
int kgs_fill_preset(kgs_ctx* ctx, int preset);

/* Page-locked host memory for fast asynchronous host<->device copies of
 * FieldState arrays (cudaHostAlloc / cudaFreeHost). */
int kgs_host_alloc(int64_t bytes, void** out);
int kgs_host_free(void* p);

/* ABI version (major*100 + minor). */
int kgs_abi_version(void);

/* Build flags of this library: KGS_BUILD_EXPERIMENTAL (-DKGS_EXPERIMENTAL:
 * the slower fused one-march step, march variants 2, 3, 5..15 and
 * kgs_debug_pass,
 * kept for the DESIGN.md §5 measurements) and KGS_BUILD_CHECKED
 * (-DKGS_CHECKED: in-kernel index asserts).  The default library has
 * neither. */
/* CUDA devices visible to this process (cudaGetDeviceCount; 0 without a
 * driver) -- ExecutorConfig("cuda", workers) uses one slab per GPU when
 * workers <= this, virtual slabs on device 0 otherwise. */
int kgs_device_count(void);

#define KGS_BUILD_EXPERIMENTAL 1
#define KGS_BUILD_CHECKED 2
int kgs_build_flags(void);

#ifdef __cplusplus
}
#endif

#endif /* KGS_B200_H */
