/* include/csc.h -- C ABI of the B200-native stochastic spatial-domain CSC hot path.
 *
 * Method: arxiv 1909.00145 ("Stochastic Convolutional Sparse Coding"), PAPER.md.
 * Citations "P:n" are PAPER.md line numbers with section/equation; readings
 * R1..R9 and #1..#17 are listed in DESIGN.md §3.
 *
 * Problem (Eq.1):  min_{d,z} sum_n 1/2||x_n - sum_k d_k * z_{n,k}||^2
 *                                       + lambda sum_{n,k} ||z_{n,k}||_1,  ||d_k||_2 <= 1.
 *
 * LAYOUTS (all row-major, contiguous, fp32, 16-byte aligned device pointers):
 *   x  [n_local][H][W]                    images of THIS rank
 *   d  [K][s][s]                          filters, replicated on every rank
 *   z  [n_local][K][H+s-1][W+s-1]         codes of THIS rank (reading R3: the
 *                                         reconstruction is a "valid" true
 *                                         convolution, no circular boundary)
 *   residual r = sum_k d_k * z_k - x      [n_local][H][W], library-owned cache.
 *
 * OWNERSHIP: x, d, z are caller-owned DEVICE pointers (e.g. torch
 * data_ptr()).  csc_code_step mutates z in place, csc_filter_step mutates d in
 * place.  The library owns the scratch of the hot path, allocated once in csc_init.
 *
 * CUDA GRAPHS: csc_zero_codes, csc_code_step and csc_filter_step with step_used == NULL
 * enqueue kernels and device-to-device work only (no allocation, no host synchronisation,
 * no pageable copy) and may be captured on dims.stream once each kernel has run once
 * (tests/test_gpu_graph.py).  The residual-cache decisions are taken on the host while
 * capturing, so a captured sequence must be replayed from the state it was captured in (e.g.
 * a SOCSC step: zero codes, code steps, filter step; or a whole iteration with
 * csc_objective_enqueue; or a streaming step with csc_load_staged in front).  csc_objective,
 * csc_iterate and any call with a host output synchronise and are not capturable;
 * csc_code_step_admm, the BCD and surrogate updates, csc_stage_images and
 * csc_iterate_staged_async allocate on first use.
 *
 * ASYNCHRONY: everything is enqueued on dims.stream (a cudaStream_t).  Only
 * csc_objective, csc_iterate(_staged), csc_objective_read, csc_iterate_drain and a non-NULL
 * step_used pointer synchronise; csc_iterate_staged_async waits for the PREVIOUS iteration only.
 *
 * COLLECTIVES (world > 1): every rank must call csc_filter_step, csc_objective
 * and csc_iterate in the same order; csc_code_step is rank-local.  The mask is a
 * counter-based function of (seed, iter, k, u, v), identical on every rank with
 * no communication.
 *
 * ERRORS: every call returns csc_status.  Argument violations return
 * CSC_ERR_ARG and have no side effects; csc_last_error(ctx) gives a message.
 * There is NO CPU fallback: without a CUDA device csc_init fails with
 * CSC_ERR_CUDA.
 *
 * RESIDUAL CACHE: the library caches r with the (x, d, z) pointers it was
 * computed from.  A different pointer, or csc_invalidate, forces a dense
 * recompute.  A caller that modifies x/d/z outside the API must call
 * csc_invalidate.
 */
#ifndef CSC_H_
#define CSC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSC_ABI_VERSION 1

typedef enum {
  CSC_OK = 0,
  CSC_ERR_ARG = 1,       /* invalid argument (no side effects) */
  CSC_ERR_SHAPE = 2,     /* unsupported shape (e.g. filter size not compiled) */
  CSC_ERR_CUDA = 3,      /* CUDA runtime error (message in csc_last_error) */
  CSC_ERR_NCCL = 4,      /* NCCL error or NCCL not loadable for world > 1 */
  CSC_ERR_OOM = 5,       /* device allocation failed in csc_init */
  CSC_ERR_NONFINITE = 6  /* a reduced scalar (objective, step) is not finite */
} csc_status;

typedef struct csc_ctx csc_ctx; /* opaque; one per (rank, device, stream) */

typedef struct {
  int32_t n_local;          /* images on this rank, >= 0 */
  int32_t K;                /* filters, >= 1 */
  int32_t s;                /* filter side, odd, 1 <= s <= 11 (compiled set: 1,3,5,7,9,11) */
  int32_t H, W;             /* image size, H >= s, W >= s; codes are K x (H+s-1) x (W+s-1) */
  int32_t world, rank;      /* world in {1,2,4,8}; 0 <= rank < world */
  int32_t device;           /* CUDA device ordinal */
  void* stream;             /* cudaStream_t (0 = legacy default stream) */
  const uint8_t* nccl_id;   /* 128-byte ncclUniqueId from csc_nccl_unique_id on rank 0,
                               broadcast by the caller; NULL when world == 1 */
} csc_dims;

/* Create a context: validates dims, binds device+stream, allocates scratch, and
 * (world > 1) joins the NCCL communicator.  *out is set only on CSC_OK. */
csc_status csc_init(const csc_dims* dims, csc_ctx** out);

/* One masked proximal-gradient step on the codes (reading R1), Eq.2-4
 * with readings R2 (unsampled codes keep their value),
 * R4/R5 (i.i.d. Bernoulli(p) per code coordinate, one mask per iteration shared
 * by all images, counter-based Philox4x32-10 generated in-kernel):
 *   for every image n and every (k,u,v) with mask bit 1:
 *     c = sum_{a,b} d[k,a,b] r[n, u-s+1+a, v-s+1+b]     (r == 0 outside the image)
 *     z[n,k,u,v] <- S_{tau*lambda}(z[n,k,u,v] - tau*c)  (shrinkage)
 * lambda >= 0; step_z > 0 is used as tau, step_z == 0 selects tau = 1/L_D(d)
 * (reading R8: L_D = max over the 64x64 DFT grid of sum_k |d_k^|^2); 0 < p <= 1;
 * iter is the mask counter t.  step_used (HOST, nullable) receives tau (syncs). */
csc_status csc_code_step(csc_ctx* ctx, const float* x, const float* d, float* z, float lambda,
                         float step_z, double p, uint64_t seed, uint32_t iter, float* step_used);

/* One projected-gradient step on the filters (reading R6) for Eq.5:
 *   g = sum_n Z_n^T (Z_n d - x_n)  (all-reduced over ranks, fp64)
 *   tau = step_d > 0 ? step_d : <g,g>/||Z g||^2  (exact line search, R8; 0 if ||Zg|| = 0)
 *   d_k <- (d_k - tau g_k) / max(1, ||d_k - tau g_k||_2)  (unit ball, R7)
 * Collective.  step_used (HOST, nullable) receives tau (syncs). */
csc_status csc_filter_step(csc_ctx* ctx, const float* x, float* d, const float* z, float step_d,
                           float* step_used);

/* Eq.1 objective over ALL ranks' images: out[0] = F,
 * out[1] = 1/2||Dz - x||^2, out[2] = lambda*||z||_1 (fp64, HOST).  Refreshes the
 * residual cache.  Collective; synchronises the stream. */
csc_status csc_objective(csc_ctx* ctx, const float* x, const float* d, const float* z,
                         float lambda, double out[3]);

/* csc_objective in two halves.  csc_objective_enqueue enqueues the objective pass (the dense residual
 * pass, which refreshes the residual cache, its reductions and, world > 1, their all-reduce) and a copy
 * of the resulting device scalars into the context's pinned host mirror, without synchronising: it may
 * be captured in a CUDA graph together with csc_code_step / csc_filter_step (one whole iteration, the
 * mask iteration supplied through csc_set_iter_offset).  csc_objective_read synchronises the stream and
 * returns out[3] as csc_objective for the last enqueued pass.  Collective (enqueue). */
csc_status csc_objective_enqueue(csc_ctx* ctx, const float* x, const float* d, const float* z);
csc_status csc_objective_read(csc_ctx* ctx, float lambda, double out[3]);

/* One SBCSC outer iteration (Alg.1): [x_host -> x upload] ->
 * csc_code_step(iter) -> csc_filter_step -> csc_objective.  When the residual cache
 * holds D z - x for the same (x, d, z) pointers, the upload moves it to the new images
 * elementwise (r <- r + x_old - x_new) instead of recomputing it.  x_host (HOST,
 * nullable, ideally pinned) is copied into the device buffer x first (the step's
 * input for the end-to-end measurement); obj_out[3] (HOST) as csc_objective;
 * taus_out[2] (HOST, nullable) = {tau_z, tau_d}.  Collective. */
csc_status csc_iterate(csc_ctx* ctx, const float* x_host, float* x, float* d, float* z,
                       float lambda, float step_z, float step_d, double p, uint64_t seed,
                       uint32_t iter, double obj_out[3], float taus_out[2]);

/* ADMM code update of the paper (§3.2), in place of the
 * one-step prox-gradient csc_code_step.  Per image n, with M = mask(seed, iter, p) (Eq.2),
 * A = D M^T and b = x_n - D z_n|off M, the selected codes w solve the masked LASSO (Eq.3)
 *   min_w 1/2||A w - b||^2 + lambda ||w||_1
 * by n_admm iterations of scaled over-relaxed ADMM started at w = y = z_n[M], u = 0:
 *   w <- n_cg conjugate-gradient steps (warm start) on (A^T A + rho I) w = A^T b + rho (y - u)
 *   w^ = alpha w + (1 - alpha) y;  y <- S_{lambda/rho}(w^ + u);  u <- u + w^ - y
 * and z_n[M] <- y; codes off M are untouched (readings A1-A6).  rho = 0 selects
 * rho = 10 lambda.  Requires lambda > 0, rho >= 0, 0 < alpha < 2, n_admm >= 1,
 * n_cg >= 1, 0 < p <= 1.  Rank-local (images are independent).  Scratch (7 code-sized fp32
 * buffers + mask bits) is allocated on the first call and kept; it is the only call that
 * allocates, so capture it in a graph only after one warm-up call. */
csc_status csc_code_step_admm(csc_ctx* ctx, const float* x, const float* d, float* z, float lambda,
                              float rho, float alpha, int n_admm, int n_cg, double p, uint64_t seed,
                              uint32_t iter);

/* Built-in code step-size rule, used by csc_code_step / csc_iterate when step_z == 0:
 *   CSC_STEP_LIPSCHITZ (default): tau = 1/L_D for every code (reading R8);
 *   CSC_STEP_ESO: tau_k = 1/(p L_D + (1-p) ||d_k||^2) for the codes of filter k -- the
 *     parallel-coordinate-descent step whose expected separable overapproximation holds for
 *     independent Bernoulli(p) sampling (E1).
 *     Equal to the Lipschitz rule at p = 1.  step_used then receives tau_0.  The ESO is derived for
 *     independent per-code sampling: csc_code_step returns CSC_ERR_ARG for ESO with CSC_MASK_SECTOR8.
 * Per context; CSC_ERR_ARG for an unknown rule. */
typedef enum { CSC_STEP_LIPSCHITZ = 0, CSC_STEP_ESO = 1 } csc_step_rule;
csc_status csc_set_step_rule(csc_ctx* ctx, int rule);

/* Mask sampling (reading R4 / DESIGN.md E5):
 *   CSC_MASK_ENTRY (default): i.i.d. Bernoulli(p) per code coordinate (Eq.2);
 *   CSC_MASK_SECTOR8: one Bernoulli(p) draw per aligned block of 8 consecutive coordinates
 *     l = (k*Hc+u)*Wc+v (one 32-B sector of fp32 codes) -- SURVEY.md §8f NEXT-4 (ii), a labelled
 *     DEVIATION from the per-entry sampling of the paper.
 * Applies to csc_code_step / csc_iterate and csc_mask_bits; csc_code_step_admm requires ENTRY. */
typedef enum { CSC_MASK_ENTRY = 0, CSC_MASK_SECTOR8 = 1 } csc_mask_mode;
csc_status csc_set_mask_mode(csc_ctx* ctx, int mode);

/* Device-side mask-iteration offset for CUDA-graph replays of a stream of steps: with offset_dev set
 * (DEVICE uint32, NULL to clear), the code step's mask uses iteration iter + *offset_dev, read on the
 * device when the mask kernel runs (a graph captured once is replayed with a new offset written into
 * offset_dev between replays; SOCSC mask iterations 10 s + i, reading #14).  The test hooks
 * (csc_mask_bits, csc_mask_selwords) and the ADMM solver ignore it.  CSC_ERR_ARG for a misaligned pointer. */
csc_status csc_set_iter_offset(csc_ctx* ctx, const uint32_t* offset_dev);

/* Test hook: the K step sizes tau_z of the last code step (DEVICE fp32 [K]; the same value K
 * times unless that step used the ESO rule). */
csc_status csc_read_step_z(csc_ctx* ctx, float* tau_dev);

/* Projected block-coordinate descent on the filters (§3.2; SURVEY.md §8f NEXT-3;
 * DESIGN.md §11, readings B1-B4), in place of the one-step csc_filter_step.  Per sweep, for
 * k = 0..K-1 in order, with the other filters fixed, the Eq.5 quadratic in d_k is minimised exactly
 *   C_kk = sum_n Z_nk^T Z_nk,  g_k = sum_n Z_nk^T (Z_n d - x_n)  (all ranks),
 *   d_k <- P_ball(d_k - (C_kk + 1e-10 tr(C_kk)/M I)^-1 g_k),  P_ball(e) = e / max(1, ||e||)
 * and the residual is updated with the change.  A filter whose codes are all zero is left
 * unchanged (flags_out[k] = 1; flags_out is a HOST array of K bytes or NULL).  sweeps >= 1 (the
 * paper uses one, warm-started).  Requires s*s <= 128.  Collective (one all-reduce of the Gram
 * blocks per sweep and one of g_k per filter).  Scratch (K*(splits+1)*M*M doubles) is allocated on
 * the first call. */
csc_status csc_filter_step_bcd(csc_ctx* ctx, const float* x, float* d, const float* z, int sweeps,
                               uint8_t* flags_out);

/* Online dictionary learning surrogates (§3.3, Eq.7-8; SURVEY.md §8f NEXT-2;
 * DESIGN.md §12).  The context keeps C (K x K blocks of M x M, fp64, 8 K^2 M^2 bytes -- 18.7 GB at
 * K = 400, s = 11) and B (K x M, fp64) and the count t:
 *   csc_surrogate_reset:   C = 0, B = 0, t = 0 (allocates on first use).
 *   csc_surrogate_update:  with the current mini-batch (x, z of this rank; all ranks together),
 *       t <- t + 1,  C <- ((t-1)/t) C + (1/t) sum_n Z_n^T Z_n,  B <- ((t-1)/t) B + (1/t) sum_n Z_n^T x_n.
 *       Collective.
 *   csc_filter_step_surrogate:  Eq.8, min 1/2 d^T C d - d^T B s.t. ||d_k|| <= 1, by projected
 *       block-coordinate sweeps (as csc_filter_step_bcd with the surrogate in place of the data).
 *       Rank-local (C, B are identical on every rank); flags_out as csc_filter_step_bcd.
 *   csc_read_surrogate:  test hook, copies C / B (DEVICE, nullable) and returns t (HOST, nullable). */
csc_status csc_surrogate_reset(csc_ctx* ctx);
csc_status csc_surrogate_update(csc_ctx* ctx, const float* x, const float* z);
csc_status csc_filter_step_surrogate(csc_ctx* ctx, float* d, int sweeps, uint8_t* flags_out);
csc_status csc_read_surrogate(csc_ctx* ctx, double* C_dev, double* B_dev, int64_t* t_out);

/* Double-buffered image input for streaming use.  csc_stage_images starts an asynchronous copy
 * of x_host (HOST, pinned, n_local*H*W floats) into the library's staging slot (0 or 1) on an
 * internal copy stream and returns at once; csc_iterate_staged(slot, ...) is csc_iterate with the
 * images taken from that slot (waiting for its copy on the device, then a device-to-device copy
 * into x).  Staging the next batch before calling csc_iterate_staged on the current one overlaps
 * the host-to-device transfer with the iteration.  A slot is reusable once the iteration that
 * consumed it has been enqueued.  CSC_ERR_ARG for an unstaged slot. */
csc_status csc_stage_images(csc_ctx* ctx, const float* x_host, int slot);
csc_status csc_iterate_staged(csc_ctx* ctx, int slot, float* x, float* d, float* z, float lambda,
                              float step_z, float step_d, double p, uint64_t seed, uint32_t iter,
                              double obj_out[3], float taus_out[2]);

/* Pipelined csc_iterate_staged for streaming use: enqueues the iteration on the staged slot and returns
 * at once with, in obj_prev / taus_prev (host), the objective {F, 1/2||r||^2, lambda||z||_1} and step sizes
 * {tau_z, tau_d} of the PREVIOUS call, waiting only for that one (*have_prev = 1; 0 on the first call
 * after csc_iterate_drain or csc_init).  The device therefore always has the next iteration queued while
 * the host reads a result.  csc_iterate_drain waits for the last enqueued iteration and returns its
 * values (*have = 0 when none is pending).  Same arithmetic and kernels as csc_iterate_staged; results
 * are identical.  Allocates two pinned result slots on first use.  obj_prev / taus_prev may be NULL. */
csc_status csc_iterate_staged_async(csc_ctx* ctx, int slot, float* x, float* d, float* z, float lambda,
                                    float step_z, float step_d, double p, uint64_t seed, uint32_t iter,
                                    double obj_prev[3], float taus_prev[2], int* have_prev);
csc_status csc_iterate_drain(csc_ctx* ctx, double obj[3], float taus[2], int* have);

/* The image half of csc_iterate_staged on its own, for CUDA-graph capture of a streaming step: enqueues
 * on the library stream a wait for the slot's latest csc_stage_images copy, x <- the slot's images and,
 * when the residual cache holds D z - x for this x, r <- r + x_old - x_new (no dense pass); then marks
 * the slot free.  Inside a capture the wait and the mark are external event nodes, so each replay
 * follows the slot's most recent staging.  Follow with csc_code_step / csc_filter_step /
 * csc_objective_enqueue (the mask iteration through csc_set_iter_offset).  CSC_ERR_ARG for a slot
 * that was never staged. */
csc_status csc_load_staged(csc_ctx* ctx, int slot, float* x);

/* Forget the residual cache (caller changed x, d or z outside the API). */
csc_status csc_invalidate(csc_ctx* ctx);

/* SOCSC (Alg.2) fresh mini-batch: z <- 0 and r <- -x exactly, no dense pass. */
csc_status csc_zero_codes(csc_ctx* ctx, const float* x, float* z);

csc_status csc_destroy(csc_ctx* ctx);

/* Last error message of ctx (or of the last failed csc_init when ctx is NULL). */
const char* csc_last_error(const csc_ctx* ctx);

/* ncclGetUniqueId into out[128] (rank 0, before csc_init with world > 1). */
csc_status csc_nccl_unique_id(uint8_t out[128]);

int csc_abi_version(void);

/* ---- test hooks (parity) ---- */

/* Mask of iteration iter in the canonical layout: bit l = (k*Hc+u)*Wc+v lives in
 * word l>>5 at bit l&31 (LSB first); ceil(K*Hc*Wc/32) words into bits_dev (DEVICE).
 * Bit = Philox4x32-10(ctr={q lo, q hi, iter, 0x4353434D}, key={seed lo, seed hi})[l&3]
 *       < floor(p*2^32), q = l>>2. */
csc_status csc_mask_bits(csc_ctx* ctx, uint32_t iter, double p, uint64_t seed, uint32_t* bits_dev);

/* The mask exactly as the tensor-core code step consumes it (selection words, the hot path's own
 * mask kernel): info[4] (HOST) receives {nkg, wper, wnc, KC}; words_dev (DEVICE, NULL to query only)
 * receives nkg*wper*Hc*Wc 32-bit words with bit i of word (kg*wper + b)*Hc*Wc + u*Wc + v equal to
 * the canonical mask bit of filter k = kg*KC + b*wnc + i (zero for k >= min(K, (kg+1)*KC)).
 * CSC_ERR_SHAPE when this context's code step does not run on the tensor cores. */
csc_status csc_mask_selwords(csc_ctx* ctx, uint32_t iter, double p, uint64_t seed, uint32_t* words_dev,
                             int32_t info[4]);

/* The context's device scalars after the last steps (HOST out[4], syncs): out[0] = sum r^2 of the last
 * residual pass (csc_objective: 2 x the fit term), out[1] = ||z||_1 of the last objective pass,
 * out[2] = ||Z g||^2 of the last filter step or csc_zg_sumsq, out[3] = <g, g> -- all over every rank's
 * images after the all-reduce (this rank's images when world == 1).  Test hook for the sharded
 * decomposition (tests/test_gpu_sharded.py). */
csc_status csc_read_scalars(csc_ctx* ctx, double out[4]);

/* ||sum_k g_k * z_k||^2 over this rank's images for a given filter-shaped g (DEVICE fp64 [K][s][s]) --
 * the local part of the line-search denominator of csc_filter_step, with no all-reduce; read it with
 * csc_read_scalars (out[2]).  Overwrites the cached gradient (csc_read_grad then returns g).  Test hook. */
csc_status csc_zg_sumsq(csc_ctx* ctx, const float* z, const double* g_dev);

/* Copy the cached residual [n_local][H][W] into r_dev (DEVICE). */
csc_status csc_read_residual(csc_ctx* ctx, float* r_dev);

/* Copy the last all-reduced filter gradient [K][s][s] (fp64) into g_dev (DEVICE). */
csc_status csc_read_grad(csc_ctx* ctx, double* g_dev);

/* L_D(d) (reading R8) computed on the device; result to *out (HOST, syncs). */
csc_status csc_lipschitz(csc_ctx* ctx, const float* d, double* out);

/* ---- observability (per-iteration trace; the Fig.1 caption's time per iteration and
 * objective) ---- */

/* Number of nonzero entries of v (DEVICE fp32, n entries) -> *count (HOST, syncs).  One counting kernel
 * on the context stream (the codes' nnz column of the per-iteration trace); not on the iteration path. */
csc_status csc_count_nonzero(csc_ctx* ctx, const float* v, int64_t n, uint64_t* count);

/* NVTX ranges ("csc_code_step", "csc_filter_step", "csc_objective", "csc_iterate", ...) around every
 * entry point of this context when enable != 0 (header-only NVTX v3: no cost without an attached tool).
 * Also switched on at csc_init by the environment variable CSC_NVTX=1. */
csc_status csc_set_nvtx(csc_ctx* ctx, int enable);

/* Poll the NCCL communicator for an asynchronous error (ncclCommGetAsyncError): CSC_OK when none (or
 * world == 1), CSC_ERR_NCCL with the NCCL error string in csc_last_error otherwise.  A rank whose peer
 * died sees the failure here instead of hanging in the next all-reduce's synchronisation; call it
 * between iterations (it does not synchronise the stream). */
csc_status csc_comm_check(csc_ctx* ctx);

/* Number of kernel launches this context has enqueued (for bench accounting). */
uint64_t csc_launch_count(const csc_ctx* ctx);

/* ---- profiling (CUDA events around every launch, on the context stream) ---- */
typedef enum {
  CSC_K_CONV = 0,          /* dense pass: residual / Zg convolution (conv_fwd_kernel) */
  CSC_K_CONV_FINALIZE = 1, /* k-split partial sum + reduction */
  CSC_K_WGRAD = 2,         /* filter-gradient correlation (wgrad_kernel) */
  CSC_K_CODE_STEP = 3,     /* masked prox-gradient code step (code_step_kernel) */
  CSC_K_MASK = 4,          /* Philox mask generation */
  CSC_K_LIPSCHITZ = 5,     /* DTFT bound */
  CSC_K_SMALL = 6,         /* reductions, step size, update/projection */
  CSC_K_ADMM = 7,          /* ADMM solver: masked D^T and CG / ADMM vector kernels */
  CSC_K_BCD = 8,           /* block-coordinate filter update: Gram, inverse, per-filter kernels */
  CSC_K_NCLASS = 9
} csc_kernel_class;

/* Enable (1) / disable (0) per-launch event timing; enabling resets the totals. */
csc_status csc_profile_enable(csc_ctx* ctx, int enable);

/* Add the elapsed times of the event pairs recorded so far to the per-class totals and keep the pairs
 * (syncs the stream).  For CUDA graphs captured while profiling was enabled: every replay re-records the
 * captured events, so calling this after each replay accumulates each replay's kernel times. */
csc_status csc_profile_sample(csc_ctx* ctx);

/* Which kernel classes are timed while profiling is enabled: bit c = csc_kernel_class c (default: all).
 * Each timed launch records two CUDA events on the context stream; timing only the long kernels keeps
 * that host-side cost out of a timed loop (launches of untimed classes still count). */
csc_status csc_profile_set_classes(csc_ctx* ctx, uint32_t class_mask);

/* Synchronises the stream, then returns the accumulated device time (ms) and the
 * number of launches of kernel class cls since csc_profile_enable(ctx, 1). */
csc_status csc_profile_read(csc_ctx* ctx, int cls, double* total_ms, uint64_t* launches);

/* Which sm_100a kernel variant this context runs (bit set = tensor-core variant):
 *   bit 0  dense passes (residual, ||Zg||^2, objective) on tcgen05 3xTF32 (csc_tc.cu)
 *   bit 1  filter gradient Z^T r on tcgen05 3xTF32 (csc_wgrad_tc.cu)
 *   bit 2  masked code step as tcgen05 3xTF32 dense-then-mask (csc_code_tc.cu)
 *   bit 3  the dense passes use the TMA-fed shared-memory-operand kernel (csc_conv_ss.cu)
 *   bit 4  the dense passes use the fp16-split TMA-fed kernel (csc_conv_h.cu, T6)
 *   bit 5  the code step uses the fp16-split kernel with TMA-fed code tiles (csc_code_h.cu)
 *   bit 6  the filter gradient uses the fp16-split kernel at the fp16 rate (csc_wgrad_h.cu)
 * The choice is fixed at csc_init from the shape (and CSC_DENSE_PATH / CSC_WGRAD_PATH /
 * CSC_CODE_PATH = simt; CSC_WGRAD_PATH = tf32 selects the 3xTF32 filter gradient). */
uint32_t csc_kernel_variants(const csc_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* CSC_H_ */
