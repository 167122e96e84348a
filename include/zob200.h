/*
 * zob200.h -- C ABI of libzob200.so, the B200-native LoZO/MeZO step engine.
 *
 * The reference (`zoserve`, /root/reference/pkg/src/zoserve) is a Python
 * package with no FFI; its drop-in seams are Python callables.  Each entry
 * below names the reference interface it replaces (file:line).  The Python
 * package paper_2605_28760_b200 binds these with ctypes and re-exposes the
 * reference's own API (lozo_step, factorized_step, estimate_coefficient,
 * forward_score, run_serving_path, sample_gaussian, digests).
 *
 * Conventions
 *   - every entry returns ZO_OK (0) or an error code; zo_last_error() gives the
 *     message of the calling thread's last failure.  Codes map to the
 *     reference exceptions: ZO_ERR_CONFIG -> ConfigError, ZO_ERR_DIMENSION ->
 *     DimensionError, ZO_ERR_INPUT -> InputError (numerics.py:40-49),
 *     ZO_ERR_ABORT -> ScoringAbort (runtime.py:147).
 *   - device state is ctx-owned; host pointers are borrowed for the call.
 *   - calls are stream-ordered on the ctx stream (zo_set_stream); entries that
 *     return host values synchronize that stream.
 *   - one ctx per device, not thread-safe (the reference's single-writer
 *     contract, adapter.py:143-146); the digest entry points are thread-safe.
 */
#ifndef ZOB200_H
#define ZOB200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZO_OK 0
#define ZO_ERR_CONFIG 1
#define ZO_ERR_DIMENSION 2
#define ZO_ERR_INPUT 3
#define ZO_ERR_ABORT 4
#define ZO_ERR_CUDA 5
#define ZO_ERR_INTERNAL 6

/* operand precision of the tensor-core scorer */
#define ZO_PREC_FP16 0
#define ZO_PREC_BF16 1
/* the reference's "real32" (model.py:149-154): the float32 forward, computed on the
 * tensor cores as 3xTF32 split GEMMs (kind::tf32, fp32 accumulate) with fp32 LN,
 * attention, GELU and loss -- the parity mode; 12 extra bytes per weight */
#define ZO_PREC_FP32 2

#define ZO_EST_LOZO 0       /* "lozo_lazy"          zo_engine.py:368 */
#define ZO_EST_FACTORIZED 1 /* "factorized_sqrt_r"  zo_engine.py:420 */
#define ZO_EST_DENSE 2      /* "dense_mezo"         zo_engine.py:476 -- materialising loop only */

/* ZoConfig.scope (zo_engine.py:79, 256-260): "lora_only" perturbs the 2-D params
 * through rank-r slots; "full" also probes every 1-D param (LN scale / shift)
 * densely with Role.DENSE_Z directions (VectorProbe, zo_engine.py:269-295). */
#define ZO_SCOPE_LORA_ONLY 0
#define ZO_SCOPE_FULL 1

/* decoder architecture.  ZOSERVE: the reference's model (model.py:170-199: GELU-tanh
 * FFN, sinusoidal positions, no biases).  OPT: the OPT family's decoder (ReLU FFN,
 * learned positions at offset 2, biases on qkv / attn_out / ff_up / ff_down,
 * pre-LN) -- the §8(f) f4 variant that real OPT checkpoints load into; its extra
 * params are the 2-D "pos_embed" [max_pos + 2, dim] and the 1-D "<blk>.<proj>.bias". */
#define ZO_ARCH_ZOSERVE 0
#define ZO_ARCH_OPT 1

typedef struct zo_ctx zo_ctx;

/* ModelConfig (model.py:62-81) + ZoConfig shape fields (zo_engine.py:71-98). */
typedef struct {
  int32_t vocab, dim, n_layers, n_heads, prompt_len;
  int32_t opt_len;   /* option token length (TaskConfig.options, model.py:328-331) */
  int32_t max_batch; /* largest per-sign batch scored in one call */
  int32_t rank;      /* ZoConfig.rank */
  int32_t estimator; /* ZO_EST_* */
  int32_t precision; /* ZO_PREC_* */
  int32_t device;
  int32_t scope;     /* ZO_SCOPE_* */
  int32_t arch;      /* ZO_ARCH_* */
  int32_t max_pos;   /* ZO_ARCH_OPT: max_position_embeddings (table rows = max_pos + 2) */
} zo_model_desc;

const char* zo_last_error(void);
int zo_version(void);

/* lifecycle */
int zo_create(zo_ctx** out, const zo_model_desc* desc);
int zo_destroy(zo_ctx* ctx);
int zo_set_stream(zo_ctx* ctx, void* cuda_stream);
int zo_synchronize(zo_ctx* ctx);
int zo_num_matrices(const zo_ctx* ctx);
/* i-th trainable matrix in sorted layer-id order (model.py:120-121 matrix_ids) */
int zo_matrix_info(const zo_ctx* ctx, int i, char* lid, int lid_cap, int64_t* rows, int64_t* cols);
int zo_device_bytes(const zo_ctx* ctx, uint64_t* bytes);

/* parameters.  init_params (model.py:84-108) regenerated on the device from the
 * Role.INIT streams, bit-exact float64 master + 16-bit operand shadows. */
int zo_init_params(zo_ctx* ctx, uint64_t init_seed, double init_scale);
int zo_upload_matrix(zo_ctx* ctx, const char* layer_id, const double* host, int64_t rows, int64_t cols);
int zo_download_matrix(zo_ctx* ctx, const char* layer_id, double* host, int64_t rows, int64_t cols);
/* 1-D params: blk{i}.ln{1,2}.{scale,shift}, ln_f.{scale,shift} (model.py:100-107) */
int zo_upload_vector(zo_ctx* ctx, const char* layer_id, const double* host, int64_t n);
/* the float64 master of a 1-D param (full scope updates it every step) */
int zo_download_vector(zo_ctx* ctx, const char* layer_id, double* host, int64_t n);

/* directions.  step_directions / lozo_direction / factorized_direction
 * (zo_engine.py:163-261): U keyed by step, V by window start (lozo) or step
 * (factorized), sampled on the device bit-exactly. */
int zo_sample_u(zo_ctx* ctx, uint64_t seed, uint64_t step);
int zo_sample_v(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu);
/* sample_gaussian(StreamKey(seed, step, layer_id, role), rows, cols) (numerics.py:161-168)
 * for an arbitrary stream; lid_hash = fnv1a64(utf8(layer_id)). */
int zo_sample_stream(zo_ctx* ctx, uint64_t seed, uint64_t step, uint64_t lid_hash, int32_t role, int64_t n,
                     double* host_out);
/* slot arenas in sorted-id order: which = 0 U (m x r), 1 V (n x r), 2 window A (m x r),
 * 3 (full scope) the 1-D params' dense directions z (n_vec x dim, sorted vector ids,
 * chained into u_digest after the matrices, zo_engine.py:256-260) */
int zo_slot_count(const zo_ctx* ctx, int32_t which, int64_t* count);
int zo_get_slot(zo_ctx* ctx, int32_t which, double* host, int64_t count);
/* asynchronous U (0) / V (1) arena snapshot into pinned host ring slot `slot` (0..3): a
 * device copy in stream order, then the host copy on a side stream overlapping the next
 * step (the host digests of run_serving_path); _wait blocks until the slot has landed and
 * returns its (engine-owned) host pointer.  A slot must be waited on before it is reused. */
int zo_slot_snapshot(zo_ctx* ctx, int32_t which, int32_t slot);
int zo_slot_snapshot_wait(zo_ctx* ctx, int32_t which, int32_t slot, const double** host);
int zo_set_slot(zo_ctx* ctx, int32_t which, const double* host, int64_t count);
/* declare which window start the V arena holds (a host upload of V leaves it
 * unknown, so the next step would fold A and resample V): resuming mid-window
 * (load_checkpoint) keeps the reference's fold schedule (runtime.py:327-330). */
int zo_set_window(zo_ctx* ctx, int64_t window_start);
/* sampler diagnostics: [short streams, exp near-ties, splice repairs] since create */
int zo_sampler_flags(zo_ctx* ctx, uint32_t flags[3]);

/* scoring.  nsign = 2: both probes (+eps, -eps) in one launch sequence, the
 * paired scorer calls of estimate_coefficient (zo_engine.py:318-326); nsign = 1:
 * a single composition (sign 0 / eval).  tokens: [B, T] prompt || option tokens,
 * gold: [nsign, B, opt_len] option tokens scored per half (model.py:239-240,
 * 261-267: with nsign = 2 and sign_mode 1 the two halves score two options of
 * one composition).  nll_out: [nsign, B]
 * per-example option NLL, float64 (model.py:202-215). */
int zo_prepare_probe(zo_ctx* ctx, double epsilon, int32_t sign_mode);
int zo_score(zo_ctx* ctx, const int32_t* tokens, const int32_t* gold, int32_t B, int32_t nsign, double* nll_out);
/* every single-token option of the task from ONE sign-0 forward (evaluate_split /
 * eval_accuracy, model.py:247-269, 444-460): the scored row prompt_len-1 never sees the
 * option token, so its logits serve all options -- per option only the loss kernel runs.
 * tokens: [B, T] (the option column is ignored), options: [n_opt] token ids, nll_out:
 * [n_opt, B].  opt_len 1 and rank <= 8 only (ZO_ERR_CONFIG otherwise: score per option). */
int zo_score_options(zo_ctx* ctx, const int32_t* tokens, const int32_t* options, int32_t n_opt, int32_t B,
                     double* nll_out);
/* canonical_mean per sign, c = (L+ - L-)/(2 eps), c_used, beta = -(lr*c_used)
 * (numerics.py:271-284, zo_engine.py:331,411,417): out4 = [L+, L-, c, beta].
 * Returns ZO_ERR_ABORT (no update armed) when a loss is not finite. */
int zo_coefficient(zo_ctx* ctx, int32_t B, double epsilon, double lr, int32_t divide_by_r, double* out4);
/* install a host-computed [L+, L-, c, beta] (custom scorer path, zo_engine.py:298-332) */
int zo_set_coefficient(zo_ctx* ctx, const double* out4);
/* accumulate_on_U for every matrix: A += beta*U (adapter.py:252-257) */
int zo_update_u(zo_ctx* ctx);
/* fold_window for every matrix (runtime.py:242-250, adapter.py:260-271): W += A V^T; A = 0 */
int zo_fold(zo_ctx* ctx);
/* factorized_step's dense update (zo_engine.py:449-450): W += (-(lr*c)/sqrt(r)) U V^T */
int zo_update_dense(zo_ctx* ctx, double lr);
/* factorized dense update mode: 0 = float64, bit-exact with the reference's axpy_outer
 * (default); 1 = tensor cores -- U V^T on tcgen05 (16-bit operands, fp32 accumulate) fused
 * into the float64-master / 16-bit-shadow read-modify-write, HBM-bound; parameters then agree
 * with the reference to ~1e-3 of each step's update, not bit for bit.  rank >= 16, % 16 == 0. */
int zo_set_update_mode(zo_ctx* ctx, int32_t mode);
/* GEMM schedule: 0 = fastest (data-parallel waves + a stream-K tail where it pays; the
 * tail's fp32 partial sums make a row's rounding depend on the per-GPU row count M);
 * 1 = row-invariant (no stream-K: every output element is one in-order tcgen05 K
 * accumulation whatever M, tile width or CTA pairing) -- the per-example NLLs of a
 * sequence are then bitwise independent of how the batch is sliced over GPUs
 * (multi-GPU exact mode sets it on every rank). */
int zo_set_schedule(zo_ctx* ctx, int32_t row_invariant);
/* full scope: every 1-D param p += (-(lr*c)) z with the installed c (VectorProbe.update,
 * zo_engine.py:290-295, 412-416); no-op for lora_only.  zo_update_dense applies it too. */
int zo_update_vectors(zo_ctx* ctx, double lr);

/* one whole lozo_step / factorized_step on the device (zo_engine.py:368-453),
 * replayed as a CUDA graph: V at window starts, U, probes, paired scoring,
 * coefficient, update.  out4 as zo_coefficient. */
int zo_step(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu, double epsilon, double lr, int32_t divide_by_r,
            const int32_t* tokens, const int32_t* gold, int32_t B, double* out4);
/* zo_step with device-resident tokens_dev [B, T] / gold_dev [B, opt_len] and no
 * host synchronisation (the fused loop a serving replica runs); results via
 * zo_read_out4.  zo_fold_async: the fold of zo_fold, stream-ordered. */
int zo_step_async(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu, double epsilon, double lr,
                  int32_t divide_by_r, const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B);
int zo_fold_async(zo_ctx* ctx);
/* zo_step_async with the step body (U sampling, probes, scoring, coefficient,
 * update) replayed as one CUDA graph; captured on first use per
 * (seed, B, epsilon, lr, divide_by_r). */
int zo_step_graph(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu, double epsilon, double lr,
                  int32_t divide_by_r, const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B);
/* the two halves of zo_step_async; multi-GPU exact mode all-gathers the
 * per-example NLLs (zo_nll_io) between them, B_total = global batch */
int zo_step_score_async(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu, double epsilon,
                        const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B);
int zo_step_apply_async(zo_ctx* ctx, double epsilon, double lr, int32_t divide_by_r, int32_t B_total);
int zo_read_out4(zo_ctx* ctx, double* out4);
/* kernels one zo_step_graph replay launches (+ the eager step-index write), and the
 * window-start launches in front of it (V sampler, extension columns, fold) */
int zo_graph_kernel_count(zo_ctx* ctx, int32_t* per_step, int32_t* per_window);
/* q-direction mode (SURVEY.md §8(e) mode 2; no reference counterpart -- the
 * reference has no multi-query estimator): rank g of G scores
 * reference step s = macro_step*G + g (its U, V window and minibatch) at the
 * shared state and leaves [L+, L-, c, beta] in the ctx (zo_out4_io moves it to /
 * from the all-gather buffers).  zo_qdir_apply_async regenerates every U_s and
 * applies the G updates in g order from the gathered [G, 4] device array.
 * lozo needs G | nu.  G = 1 reproduces zo_step_async. */
int zo_qdir_score_async(zo_ctx* ctx, uint64_t seed, uint64_t macro_step, int32_t G, int32_t g, int32_t nu,
                        double epsilon, double lr, int32_t divide_by_r, const int32_t* tokens_dev,
                        const int32_t* gold_dev, int32_t B);
int zo_out4_io(zo_ctx* ctx, void* dev, int32_t to_ctx);
int zo_qdir_apply_async(zo_ctx* ctx, uint64_t seed, uint64_t macro_step, int32_t G, double lr,
                        const double* out4_all_dev);
/* the split steps with their bodies replayed as captured CUDA graphs (one graph launch per
 * half instead of ~370 kernel launches; the collective runs between the two launches).
 * Staging (step index, tokens, window fold / V resample) stays eager in front of the score
 * graph.  Graphs are captured on first use per (seed, B, epsilon[, lr, divide_by_r]) /
 * (B_total, epsilon, lr, divide_by_r) / (seed, G, lr, gather buffer) and dropped by
 * zo_set_update_mode / zo_set_schedule.  Results are identical to the _async forms. */
int zo_step_score_graph(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu, double epsilon,
                        const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B);
int zo_step_apply_graph(zo_ctx* ctx, double epsilon, double lr, int32_t divide_by_r, int32_t B_total);
int zo_qdir_score_graph(zo_ctx* ctx, uint64_t seed, uint64_t macro_step, int32_t G, int32_t g, int32_t nu,
                        double epsilon, double lr, int32_t divide_by_r, const int32_t* tokens_dev,
                        const int32_t* gold_dev, int32_t B);
int zo_qdir_apply_graph(zo_ctx* ctx, uint64_t seed, uint64_t macro_step, int32_t G, double lr,
                        const double* out4_all_dev);
/* kernels per launch of [score, apply, qdir score, qdir apply] graphs (0 before capture) */
int zo_split_graph_kernels(zo_ctx* ctx, int32_t out[4]);
/* materialising training-loop comparand (baseline_loop.py:122-239, run_baseline;
 * replaces the _Probe / VectorProbe writes of baseline_loop.py:68-119, 191-221):
 * zo_baseline_directions samples the step's U (+ V at a window start / every
 * factorized step) and zeroes the LoRA-extension operands (the forward reads the
 * materialised weights); zo_baseline_pass writes the probe into the weights --
 * pass 0: +eps P, 1: -2 eps P, 2: restore (recompute = 0: cached product, the
 * restore copies the saved bits; 1: axpy_outer recompute, arithmetic restore) --
 * with zo_score(nsign = 1) in between; zo_baseline_update applies
 * W += (beta*scale) P with the ctx coefficient (zo_coefficient / zo_set_coefficient).
 * zo_baseline_step_async: one whole step, device inputs, no host sync. */
int zo_baseline_directions(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu);
int zo_baseline_pass(zo_ctx* ctx, int32_t pass, double epsilon, int32_t recompute);
int zo_baseline_update(zo_ctx* ctx, double lr, int32_t recompute);
int zo_baseline_step_async(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu, double epsilon, double lr,
                           int32_t divide_by_r, int32_t recompute, const int32_t* tokens_dev,
                           const int32_t* gold_dev, int32_t B);
/* per-phase device time of the last zo_step (ms): [sample, score, update] */
int zo_last_step_ms(zo_ctx* ctx, float ms[3]);

/* FNV-1a-64 (numerics.py:60-124), chained from h.  Thread-safe, host only. */
uint64_t zo_fnv1a64(const void* data, uint64_t nbytes, uint64_t h);
/* u/v digest chain over sorted layer ids (zo_engine.py:220-261) of a host copy of
 * an arena: for i: h = fnv(lid_i); h = fnv(arena[off_i : off_i + cnt_i]) */
uint64_t zo_digest_chain(const char* const* lids, const double* arena, const int64_t* offsets,
                         const int64_t* counts, int32_t n, uint64_t h);

/* measurement: average ms of one launch of a layer GEMM at batch B
 * (which: 0 qkv, 1 attn_out, 2 ff_up, 3 ff_down, 4 LM head) and its FLOPs */
int zo_bench_gemm(zo_ctx* ctx, int32_t which, int32_t B, int32_t reps, float* avg_ms, double* flops);
/* one eager zo_step_async (device inputs, divide_by_r = 0) with a CUDA event in front of every
 * scorer kernel group; ms[10] = device ms per family summed over the layers: embed, LN, qkv GEMM,
 * attention, extension finalize, attn_out GEMM, ff_up GEMM, ff_down GEMM, last-layer tail + LM
 * head + loss, other (sampler, probes, coefficient, update).  The bench's in-step roofline. */
/* diagnostic timeline of one launch of a layer GEMM (which as zo_bench_gemm): per CTA 64
 * globaltimer stamps -- [0] start, [1] end, [2+2i, 3+2i] MMA window and [32+2i, 33+2i]
 * epilogue window of the CTA's i-th tile segment (i < 15); *grid = the launch's CTA count */
int zo_trace_gemm(zo_ctx* ctx, int32_t which, int32_t B, uint64_t* host, int32_t cap, int32_t* grid);
int zo_profile_step(zo_ctx* ctx, uint64_t seed, uint64_t step, int32_t nu, double epsilon, double lr,
                    const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B, float* ms);
/* copy per-example NLLs between the ctx and an external device buffer
 * (to_ctx = 1: dev -> ctx) -- the multi-GPU exact-mode exchange point */
int zo_nll_io(zo_ctx* ctx, void* dev, int32_t count, int32_t to_ctx);

/* test hook: D = A[M,K] . B[N,K]^T through the production tcgen05 GEMM with
 * epilogue epi (0 store16, 1 gelu16, 2 resid32: C += D, 3 store32); host
 * buffers, 16-bit inputs with row stride lda, fp32 output [M, N]. */
int zo_test_gemm(int32_t M, int32_t N, int32_t K, int32_t lda, int32_t epi, int32_t bf16, const uint16_t* A_host,
                 const uint16_t* B_host, float* C_host);

/* test hook of the real32 path: C[M, N] = A[M, K] . W[K, N] (A fp32, W float64 (in, out))
 * through the 3xTF32 operand split and the tf32 tcgen05 GEMM; host buffers. */
int zo_test_gemm_tf32x3(int32_t M, int32_t N, int32_t K, const float* A_host, const double* W_host, float* C_host);

#ifdef __cplusplus
}
#endif
#endif
