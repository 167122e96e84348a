// Non-GEMM kernels of the LoZO step (scorer glue, loss, coefficient, update, fold).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace zo {

// Activation/weight operand precision for the tensor-core path.
struct H16 {
  bool bf16;
};

// learned position table (OPT arch): row t + offset of W64 [max_pos + 2, d] plus its
// LoRA delta; W64 == nullptr: the fixed sinusoidal table pe[T, d] (model.py:128-136)
struct PosEmbed {
  const double* W64 = nullptr;
  const float* Pp = nullptr;
  const float* Pm = nullptr;
  const float* V32 = nullptr;
  int offset = 0;
};
// x32[M,d] = E[tok] + sum_k P_s[tok,k] V_e[:,k] + PE[t]   (model.py:180, adapter.py:200-234)
// for positions t < T of token rows tokens[b * tok_ld + t]
// token rows from E64 (float64 master), else E32 (fp32 master), else E16 (16-bit shadow)
void launch_embed(float* x32, const int32_t* tokens, int tok_ld, int B, int T, int d, const double* E64,
                  const float* E32, const void* E16, bool bf16, const float* Pplus, const float* Pminus, const float* Ve32, int r,
                  const float* pe, const PosEmbed& pos, int nrows, cudaStream_t st);
// h = LN(x) (model.py:139-142) -> out[:, :d] (16-bit); ext columns [d, d+3r) = (t_hi, t_lo, t_hi)
// per rank with t = h . P_s (fp32) -- the LoRA K-extension operand (A side).
// vstride: offset (floats) of the -eps copy of gamma/beta read by rows >= rows_per_sign
// (full scope, 0 otherwise)
void launch_ln_ext(const float* x32, const float* gamma, const float* beta, int M, int d, void* out, int ldo,
                   bool bf16, const float* Pplus, const float* Pminus, int r, int rows_per_sign, int ext_terms,
                   long vstride, cudaStream_t st);
// ext columns for a 16-bit activation a[:, :K] already in place (ctx -> attn_out, gelu -> ff_down).
void launch_ext(void* a, int lda, int M, int K, bool bf16, const float* Pplus, const float* Pminus, int r,
                int rows_per_sign, int ext_terms, cudaStream_t st);
// Fused LoRA-extension partials of an activation producer: tpart[tile][row][k]
// (tile = head for attention), finished by launch_ext_finalize.
struct AttnExt {
  const float* Pp = nullptr;
  const float* Pm = nullptr;
  int r = 0, rps = 0, ld = 0;  // rank, rows per sign, rows per tile slab
  float* tpart = nullptr;      // nullptr: no fused extension
};
// causal softmax attention per (sequence, head) (model.py:184-194); qkv [M,3d] -> ctx[:, :d]
void launch_attention(const void* qkv, int ldq, void* ctx, int ldc, int nseq, int T, int H, int dh, bool bf16,
                      const AttnExt& x, cudaStream_t st);
// t_k = sum over tiles of tpart[tile][row][k] (fixed order) -> ext columns (hi, lo, hi) of a[:, K:]
void launch_ext_finalize(const float* tpart, int ntiles, int ld, int M, int r, void* a, int lda, int K,
                         int ext_terms, bool bf16, cudaStream_t st, int neg_from = -1);
// dst row i = src row of the i-th scored (sign, sequence, option token): the compact
// rows the last layer's pruned tail runs on (row_bytes, strides in bytes)
void launch_gather_scored(const void* src, size_t ld_src_bytes, void* dst, size_t ld_dst_bytes, int row_bytes,
                          int nsign, int B, int T, int prompt_len, int Lopt, cudaStream_t st);
// final LN at scored rows (prompt_len-1+j) of B sequences (both signs counted) -> xs32/xs16, z = xs . V_e
void launch_final_ln(const float* x32, const float* gamma, const float* beta, int B, int T, int d,
                     int prompt_len, int Lopt, float* xs32, void* xs16, bool bf16, const float* Ve32, int r,
                     float* z, int rows_per_sign, long vstride, cudaStream_t st);
// per scored row: logits + z.P_s,e^T -> log-softmax, gold gather -> nll[sign*B + b] (model.py:202-215);
// ws: loss_ws_floats(2*B*Lopt, V) floats, counters: 2*B*Lopt + 2*B zeroed (self-resetting)
int loss_splits(int V);
size_t loss_ws_floats(int rows, int V);
void launch_loss(const float* logits, int ldl, int V, const float* z, int r, const float* Pplus_e,
                 const float* Pminus_e, const int32_t* gold, int B, int Lopt, float* ws, unsigned* counters,
                 double* nll, cudaStream_t st);
// canonical_mean per sign, c, c_used, beta (numerics.py:271-284, zo_engine.py:331,411)
void launch_coefficient(const double* nll, int B, double eps, double lr, int divide_by_r, int rank,
                        double* out4, unsigned* abort_flag, cudaStream_t st);
// A += beta*U (numerics.py:238-243; product then sum, no FMA); skipped when aborted
void launch_update(double* A, const double* U, int64_t n, const double* out4, const unsigned* abort_flag,
                   cudaStream_t st);
// P+- = fp32(A +- eps*U)
void launch_prep_probe(const double* A, const double* U, int64_t n, double eps, double probe_scale, float* Pp,
                       float* Pm, cudaStream_t st);
// full scope (VectorProbe, zo_engine.py:269-295): out32[0] = fp32(p + eps*z), out32[1] =
// fp32((p + eps*z) + (-2 eps)*z) (both fp32(p) when eps == 0); update p += (-(lr*c))*z
void launch_vec_probe(const double* p, const double* z, int64_t n, double eps, float* out32, cudaStream_t st);
void launch_vec_update(double* p, const double* z, int64_t n, const double* out4, double lr,
                       const unsigned* abort_flag, float* out32, cudaStream_t st);
// P16T[k][i] = h16(P[i][k]) for one [m, r] probe block (tensor-core extension B operand, r > 8)
void launch_p16t(const float* P, int m, int r, void* out, bool bf16, cudaStream_t st);
// launch_p16t for every matrix of tab ({first 32-row tile, u_off, m} per matrix) and both signs
void launch_p16t_all(const float* Pp, const float* Pm, int64_t su, const int64_t* tab, int ntab, int tiles, int r,
                     int nsign, void* out, bool bf16, cudaStream_t st);
// V ext columns (hi, hi, lo) into W16T[:, K:K+3r] for one matrix; V32 copy
void launch_write_vext(const double* V, int n, int r, void* W16T, int ldw, int K, bool bf16, int ext_terms,
                       float* V32, cudaStream_t st);
// every matrix's V -> V32 (+ its W16T extension columns) in one launch; tab sorted by v_off
struct VextMat {
  int64_t v_off;
  void* W;  // W16T (nullptr: V32 only -- the embedding)
  int ldw, K;
};
void launch_write_vext_all(const double* V, int64_t sv, const VextMat* tab, int ntab, int r, bool bf16,
                           int ext_terms, float* V32, cudaStream_t st);
// W64[m,n] += sum_k A[:,k] V[:,k]^T (k ascending, numerics.py:207-235) then A = 0
void launch_fold(double* W64, int m, int n, const double* A, const double* V, int r, double alpha, void* W16,
                 int ldw, int transposed, bool bf16, cudaStream_t st);
void launch_fold_dev(double* W64, int m, int n, const double* A, const double* V, int r, const double* out4,
                     double lr, double scale, const unsigned* abort_flag, void* W16, int ldw, int transposed,
                     bool bf16, cudaStream_t st);
// shadows: W16T[n, :m] = h16(W64[m,n]^T) (projection) or E16[m, n] = h16(W64) (embed)
void launch_shadow_T(const double* W64, int m, int n, void* W16T, int ldw, bool bf16, cudaStream_t st);
void launch_shadow(const double* W64, int64_t count, void* W16, bool bf16, cudaStream_t st);
void launch_zero(void* p, size_t bytes, cudaStream_t st);
// materialising-loop comparand (baseline_loop.py:68-239): mode 0 cached probe (16-bit copy
// of fl(fl(w0 + a1*P) [+ a2*P]) only), 1 cached update (alpha = out4[3]*scale), 2 recompute
// (axpy_outer in place, alpha = a1 or out4[3]*scale); modes 1/2 write master + 16-bit copy
void launch_materialise(int mode, double* W64, int m, int n, const double* U, const double* V, int r, double a1,
                        double a2, const double* out4, double scale, void* W16, int ldw, int transposed, bool bf16,
                        cudaStream_t st);
// dense_mezo materialising loop (_DenseProbe, baseline_loop.py:107-119): the same modes with
// the dense direction Z[m, n] in place of the rank-r product (mode 3 = shadow copy)
void launch_dense_rw(int mode, double* W64, int m, int n, const double* Z, double a1, double a2, const double* out4,
                     void* W16, int ldw, int transposed, bool bf16, cudaStream_t st);
// 1-D params in place (recompute-mode _DenseProbe): p += alpha*z, alpha = a1 or out4[3]
void launch_vec_inplace(double* p, const double* z, int64_t n, double a1, const double* out4, float* out32,
                        cudaStream_t st);
// VectorProbe at one sign for a single-sign scoring call (both fp32 copies)
void launch_vec_probe_sign(const double* p, const double* z, int64_t n, double eps, int sign, float* out32,
                           cudaStream_t st);
void launch_f64_to_f32(const double* a, float* b, int64_t n, cudaStream_t st);
void launch_f32_to_f64(const float* a, double* b, int64_t n, cudaStream_t st);

}  // namespace zo
