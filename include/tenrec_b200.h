/*
 * tenrec_b200 -- C ABI of the B200 randomized t-SVT / ADMM recovery path.
 *
 * Plain pointers and sizes only (no torch types).  All tensor pointers are
 * DEVICE pointers to dense column-major arrays (first index fastest, the
 * reference's convention, tenrec/core.py:1-8).  `dtype` selects the streaming
 * precision of the large tensors: TR_F32 (float) or TR_F64 (double).  Small
 * dense algebra always runs in fp64.  `stream` is a cudaStream_t (NULL = the
 * legacy default stream).  Every call is asynchronous on `stream` unless noted
 * and returns 0 on success; a nonzero code leaves a message in
 * tr_last_error().  Workspaces are caller-owned device buffers whose size is
 * given by the matching *_workspace() query.
 *
 * Each entry point below names the reference interface it replaces.
 */
#ifndef TENREC_B200_H
#define TENREC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TR_F32 0
#define TR_F64 1

/* Transform kinds (tenrec/transform.py:44-80): FFT default, orthonormal DCT-II,
 * explicit unitary-up-to-scale matrices. */
#define TR_TRANSFORM_FFT 0
#define TR_TRANSFORM_DCT 1
#define TR_TRANSFORM_EXPLICIT 2

/* Penalty kinds (tenrec/penalties.py, make_penalty:276-290) with parameters
 * (p0, p1): l1 (-), firm (gamma), mcp (gamma), scad (a), lq (q),
 * capped-lq (q, theta), log (gamma). */
#define TR_PEN_L1 0
#define TR_PEN_FIRM 1
#define TR_PEN_MCP 2
#define TR_PEN_SCAD 3
#define TR_PEN_LQ 4
#define TR_PEN_CAPPED_LQ 5
#define TR_PEN_LOG 6

/* Library version (major*10000 + minor*100 + patch). */
int tr_version(void);

/* Message of the last failed call on this host thread. */
const char* tr_last_error(void);

/* Device workspace bytes for tr_gnhtsvt_randomized / tr_rsthosvd_bki. */
int64_t tr_lrta_workspace(int dtype, int order, const int64_t* dims, const int64_t* ranks,
                          const int64_t* blocks, const int64_t* krylov);

/*
 * Randomized GNHTSVT -- replaces tenrec.sketch.gnhtsvt_randomized
 * (tenrec/sketch.py:430-456) for a fixed-rank SketchConfig with the default
 * processing order (0, 1): block-Krylov Tucker compression of modes 0 and 1
 * (sketch.py:211-270), transform-domain singular value thresholding of the
 * core with penalty.prox(tau, .) (shrink.py:76-106), re-expansion.
 *
 *   a, out        n1 x n2 x ... x nd tensors (dtype), out may not alias a
 *   order, dims   d >= 3 and the d mode lengths
 *   ranks/blocks/krylov  two entries each (modes 0 and 1)
 *   seed          sketch seed; sketch entry (c, t) of processing step p is
 *                 N(0,1) from Philox4x32-10 at (seed, p, c*b + t)
 *   transform_kind, transform_mats, alphas
 *                 for TR_TRANSFORM_EXPLICIT: device complex128 (interleaved)
 *                 row-major matrices of the trailing modes, concatenated, and
 *                 their host scalings alpha_i; ignored otherwise
 *   penalty_kind, p0, p1, tau   the thresholding penalty and level
 *   sketch0, sketch1  optional device override of the two sketch matrices
 *                 (dtype, row-major (n2*nf) x b0 and (r0_eff*nf) x b1), used to
 *                 replay an externally drawn Gaussian stream; NULL = Philox
 */
int tr_gnhtsvt_randomized(int dtype, const void* a, void* out, int order, const int64_t* dims,
                          const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                          uint64_t seed, int transform_kind, const void* transform_mats,
                          const double* alphas, int penalty_kind, double p0, double p1,
                          double tau, const void* sketch0, const void* sketch1, void* workspace,
                          int64_t workspace_bytes, void* stream);

/*
 * Sharded randomized t-SVT (multi-GPU, one rank per GPU): this rank holds the
 * slice [last_off, last_off + dims[order-1]) of the LAST mode of a tensor whose
 * last mode has length last_all (`dims` are the LOCAL dims; earlier modes
 * whole).  The mode-0/1 Krylov partial sums, the Ritz Gram and the compressed
 * r0 x r1 x faces core are summed across ranks through `allreduce` (in place,
 * fp64, ordered on `stream`; e.g. NCCL through torch.distributed), the sketch
 * is drawn at GLOBAL column indices, so every rank's `out` slice equals the
 * same slice of the single-GPU tr_gnhtsvt_randomized result up to summation
 * order.  Workspace: tr_lrta_workspace of the GLOBAL dims.  Returns 0 / error.
 */
typedef int (*tr_allreduce_fn)(double* buf, int64_t count, void* stream, void* user);
int tr_gnhtsvt_randomized_sharded(int dtype, const void* a, void* out, int order,
                                  const int64_t* dims, int64_t last_all, int64_t last_off,
                                  const int64_t* ranks, const int64_t* blocks,
                                  const int64_t* krylov, uint64_t seed, int transform_kind,
                                  const void* transform_mats, const double* alphas,
                                  int penalty_kind, double p0, double p1, double tau,
                                  tr_allreduce_fn allreduce, void* user, void* workspace,
                                  int64_t workspace_bytes, void* stream);

/*
 * Fixed-rank Tucker compression of modes (0, 1) -- replaces
 * tenrec.sketch.rsthosvd_bki(x, ranks, order=(0, 1), ...) (sketch.py:211-270).
 * Outputs (device, fp64, zero-padded to the requested ranks):
 *   f0 n1 x r0, f1 n2 x r1, core r0 x r1 x n3 x ... x nd, ranks_eff[2] (int64).
 */
int tr_rsthosvd_bki(int dtype, const void* a, int order, const int64_t* dims,
                    const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                    uint64_t seed, const void* sketch0, const void* sketch1, double* f0,
                    double* f1, double* core, int64_t* ranks_eff, void* workspace,
                    int64_t workspace_bytes, void* stream);

/*
 * Generic Tucker compression -- replaces tenrec.sketch.rsthosvd_bki for any
 * processing order (sketch.py:211-270) and tenrec.sketch.ad_rsthosvd_blbp
 * (fixed-accuracy block Lanczos bidiagonalisation, sketch.py:287-403); with
 * tr_tucker_svt it replaces tenrec.sketch.gnhtsvt_randomized for every
 * SketchConfig the fused tr_gnhtsvt_randomized does not take (sketch.py:406-456).
 * Host-synchronous: returns once the factors and core are on the device.
 *
 *   a, order, dims   the tensor (dtype, device, column-major)
 *   sketch_mode      0 fixed-rank (ranks/blocks/krylov per processed mode),
 *                    1 fixed-accuracy (eps, block, defl_tol <= 0 for the default
 *                    1e-10 ||unfolding||_F)
 *   nproc, proc_order  the modes to compress, in processing order
 *   seed             Philox seed: fixed-rank step p draws entry (c, t) at
 *                    (seed, p, c*b + t); fixed-accuracy draw j (start block of a
 *                    mode or fill block, counted in call order across modes) is
 *                    the (n, cols) block of entries (seed, j, c*cols + t)
 * Factor columns carry the canonical sign (largest-|entry| positive).
 * tr_tucker_info: per mode (order entries) core dims, ranks (dims[k] for
 * unprocessed modes), processed flags and the BLBPDiagnostics traces (energy,
 * deflations, iterations, local orthogonality loss); any pointer may be NULL.
 * tr_tucker_read: which = -1 copies the core (fp64, natural column-major
 * layout), which = k the factor of mode k (fp64, dims[k] x ranks[k]).
 * tr_tucker_svt: out (dtype, the full dims) = the transform-domain SVT of the
 * core (transform adapted to the core's trailing sizes) re-expanded through
 * the factors; the handle's core is not modified.
 */
int tr_tucker_create(int dtype, const void* a, int order, const int64_t* dims, int sketch_mode,
                     int nproc, const int64_t* proc_order, const int64_t* ranks,
                     const int64_t* blocks, const int64_t* krylov, double eps, int64_t block,
                     double defl_tol, uint64_t seed, void* stream, void** handle);
int tr_tucker_info(void* handle, int64_t* core_dims, int64_t* ranks, int64_t* processed,
                   double* energy, int64_t* deflations, int64_t* iterations, double* orth_loss);
int tr_tucker_read(void* handle, int which, double* dst, void* stream);
int tr_tucker_svt(void* handle, int transform_kind, const void* transform_mats,
                  const double* alphas, int penalty_kind, double p0, double p1, double tau,
                  void* out, void* stream);
int tr_tucker_destroy(void* handle);

/*
 * Elementwise proximity operator -- replaces Penalty.prox(mu, v)
 * (tenrec/penalties.py:45-61) on a device array of n values (dtype).
 */
int tr_prox(int dtype, int penalty_kind, double p0, double p1, double mu, const void* v,
            void* out, int64_t n, void* stream);

/*
 * ADMM solvers -- replace tenrec.solvers.gnrhtc / gnhtc (solvers.py:204-295) and
 * tenrec.onebit.gnobhtc / gnobrhtc (onebit.py:141-234).  A solver owns its
 * device state; the caller keeps the observation buffers alive until destroy.
 *
 *   kind       0 gnrhtc (obs_a = Mobs, mask), 1 gnhtc (noise-free),
 *              2 gnobhtc (obs_a = J1, obs_b = J2), 3 gnobrhtc (robust one-bit)
 *   modes      the gradient set Gamma (0-based modes); {-1} = identity chain
 *              (the pure low-rank ablation, SolverConfig.pure_lowrank)
 *   structure  noise shrinkage groups: 0 entry, 1 tube, 2 slice
 *   phi / psi  low-rank and noise penalties (kind, p0, p1)
 *   lam, lam2  trade-off weights; mu0, mu_max, growth the penalty schedule;
 *   alpha      one-bit box bound; mcount the one-bit sample count m
 *   randomized 1 = randomized t-SVT with ranks/blocks/krylov/seed (modes 0, 1);
 *              0 = deterministic t-SVT (face slices up to 64 x 64)
 * tr_admm_step runs one sweep and writes TR_ADMM_NOUT residuals to `out`
 * (host): [dL, dE, grad_gap, dG, fit_gap, dL_fro, dE_fro, dG_fro, fit_fro,
 *  grad_gap_fro, ||Y||, max_k ||Lambda_k||, mu, rel_dL (one-bit), box_gap (one-bit)].
 * tr_admm_read copies state `which` (0 L, 1 E or S, 2 Y, 3 Z, 4 + k the G tensor of
 * gradient mode k, i.e. the last sweep's t-SVT output) to `dst` (device).
 */
#define TR_ADMM_NOUT 15
int tr_admm_create(int dtype, int order, const int64_t* dims, int kind, const void* obs_a,
                   const void* obs_b, const uint8_t* mask, int nmodes, const int64_t* modes,
                   int structure, int phi_kind, double phi_p0, double phi_p1, int psi_kind,
                   double psi_p0, double psi_p1, double lam, double lam2, double mu0,
                   double mu_max, double growth, double alpha, double mcount, int randomized,
                   const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                   uint64_t seed, int transform_kind, const void* transform_mats,
                   const double* alphas, void** handle);
int tr_admm_step(void* handle, double* out);
/* on != 0: tr_admm_step enqueues the L-solve and the t-SVT inputs of the NEXT
 * sweep before it waits for this sweep's residuals, so the GPU does not idle
 * across the host's read-back and stopping test (tenrec/solvers.py:270-272 tests
 * on the host after every iteration).  The returned state (tr_admm_read) and
 * every later residual are unchanged; a caller that stops after a step leaves
 * that work unused -- switch it off before the last step of a fixed-length
 * run.  Applies to the fused gradient chain on one GPU; ignored otherwise. */
int tr_admm_lookahead(void* handle, int on);
int tr_admm_read(void* handle, int which, void* dst, void* stream);
int tr_admm_destroy(void* handle);
/*
 * Multi-GPU ADMM (BASELINE configs[4]; north_star's sharded solve): rank `rank`
 * of `world` holds faces [last_off, last_off + dims[order-1]) of the LAST mode
 * (length last_all = world * dims[order-1]); `dims` are the local dims and
 * obs_a / mask the local slabs.  Per sweep: the FFT-diagonal L-solve runs the
 * local axes in place and the last axis after an all-to-all transpose (each
 * rank then owns whole last-axis lines of 1/world of the spectrum) and back;
 * the circular stencils along the last axis read one ghost face per
 * neighbour (halo exchange of L, the last mode's G and multiplier); every
 * t-SVT is the last-mode-sharded one of tr_gnhtsvt_randomized_sharded (fp64
 * all-reduces of the Krylov blocks, Ritz Gram and core); the Eq. (24)
 * residuals are all-reduced (sum / max) so tr_admm_step returns the global
 * values on every rank.  GNRHTC / GNHTC, entry-wise noise, randomized
 * fixed-rank sketch of modes (0, 1), FFT transform.  The collectives are the
 * caller's, ordered on `stream` (e.g. NCCL through torch.distributed):
 *   allreduce  in-place fp64 over `count` values, op 0 sum / 1 max
 *   alltoall   `bytes` from send + q*bytes go to rank q, recv + q*bytes
 *              come from rank q
 *   halo       send first_face to rank-1 and last_face to rank+1 (ring);
 *              receive rank-1's last face into ghost_prev and rank+1's first
 *              face into ghost_next (`bytes` each)
 * world == 1 needs no callbacks (the exchanges are local copies).
 */
typedef struct tr_comm {
  int world, rank;
  int (*allreduce)(double* buf, int64_t count, int op, void* stream, void* user);
  int (*alltoall)(const void* send, void* recv, int64_t bytes, void* stream, void* user);
  int (*halo)(const void* first_face, const void* last_face, void* ghost_prev, void* ghost_next,
              int64_t bytes, void* stream, void* user);
  void* user;
} tr_comm;
int tr_admm_create_sharded(int dtype, int order, const int64_t* dims, int kind,
                           const void* obs_a, const uint8_t* mask, int nmodes,
                           const int64_t* modes, int phi_kind, double phi_p0, double phi_p1,
                           int psi_kind, double psi_p0, double psi_p1, double lam, double mu0,
                           double mu_max, double growth, const int64_t* ranks,
                           const int64_t* blocks, const int64_t* krylov, uint64_t seed,
                           int64_t last_all, int64_t last_off, const tr_comm* comm,
                           void** handle);

/* Route the solver's t-SVTs through the generic Tucker engine (tr_tucker_*)
 * with this sketch: any processing order, fixed-rank (sketch_mode 0) or
 * fixed-accuracy block Lanczos (sketch_mode 1); arguments as tr_tucker_create.
 * Replaces the randomized/ranks/blocks/krylov/seed of tr_admm_create. */
int tr_admm_set_sketch(void* handle, int sketch_mode, int nproc, const int64_t* proc_order,
                       const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                       double eps, int64_t block, double defl_tol, uint64_t seed);
/* The solver's main cudaStream_t (every sweep starts and ends on it). */
void* tr_admm_stream(void* handle);

/*
 * Gradient system -- replaces tenrec.gradient.GradientSet (gradient.py:44-87)
 * and solve_grad_system (gradient.py:90-106): out = (I + sum_k D_k^T D_k)^{-1}
 * (b + sum_k D_k^T grads[k]), D_k the forward circular difference along mode
 * modes[k].  The plan holds the FFT twiddles and the eigenvalue tables
 * 4 sin^2(pi j / n); b, grads[k] (one per mode, in `modes` order) and out are
 * device arrays of prod(dims) values in the plan's dtype, first axis fastest.
 * order in [3, 8]; modes distinct.  Destroy with tr_gradsys_destroy.
 */
int tr_gradsys_create(int dtype, int order, const int64_t* dims, int nmodes, const int* modes,
                      void** handle);
int tr_gradsys_solve(void* handle, const void* b, const void* const* grads, void* out,
                     void* stream);
int tr_gradsys_destroy(void* handle);

/* Number of kernels this library has launched in the process (accounting). */
int64_t tr_launch_count(void);

/* Enable (1) / disable (0) per-category CUDA-event timing of every launch;
 * either call discards previously recorded events. */
int tr_profile_enable(int on);

/* Synchronise the recorded events and aggregate them per kernel category:
 * writes up to max_entries totals (ms) and launch counts, and the category
 * names joined by '\n' into `names`.  Returns the number of categories. */
/* Per-launch timeline of the profiled region (diagnostics; not in the reference). */
int tr_profile_timeline(char* names, int64_t names_len, double* t0, double* t1, int64_t* streams,
                        int max_entries);
int tr_profile_read(char* names, int64_t names_len, double* ms, int64_t* counts,
                    int max_entries);

#ifdef __cplusplus
}
#endif

#endif /* TENREC_B200_H */
