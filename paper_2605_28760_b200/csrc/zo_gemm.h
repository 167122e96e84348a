// K2 -- tcgen05/TMEM/TMA GEMM for the scorer's projections and LM head.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace zo {

enum EpiKind : int {
  EPI_STORE16 = 0,  // out16[r, c] = acc                       (qkv)
  EPI_GELU16 = 1,   // out16[r, c] = gelu_tanh(acc)            (ff_up, model.py:145-146,197)
  EPI_RESID32 = 2,  // x32[r, c] += acc                        (attn_out / ff_down residual)
  EPI_STORE32 = 3,  // out32[r, c] = acc                       (LM-head logits rows)
  EPI_GELU16_EXT = 4,  // EPI_GELU16 + partial t_k = sum_c a16[r,c] P[c,k] per 128-column slot
                       // for the next GEMM's LoRA K-extension (tpart[slot][r][k], deterministic)
  EPI_UPDATE64 = 5,    // factorized dense update on the tensor cores (zo_engine.py:449-450), the
                       // plan-level kind: W += alpha * acc (alpha = -(lr*c)*scale from the device
                       // coefficient, skipped when the step aborted) on an fp32 master, the
                       // 16-bit shadow rewritten in the same pass; D = V U^T (upd_transposed)
  EPI_UPDATE32 = 6,    // the kernel variant that runs EPI_UPDATE64 plans
};

// D[M, N] = A[M, Kp] * B[N, Kp]^T, both operands K-major 16-bit, fp32 accumulate.
struct GemmDesc {
  CUtensorMap tmA;
  CUtensorMap tmB;
  CUtensorMap tmB2;  // B with a half-height box: the half-width tail tiles (gemm_enable_halftail)
  CUtensorMap tmO;   // the epilogue output for TMA stores / reduce-adds (res_tma)
  int M = 0, N = 0;
  int num_kb = 0;       // 64-wide K blocks
  int last_ksteps = 4;  // 16-wide UMMA steps issued in the last K block (trims the LoRA extension)
  int bn = 256;         // tile N (64/128/256)
  int cg = 1;           // 2: CTA-pair tiles (tcgen05 cta_group::2, M = 256, B split across the pair)
  int epi = EPI_STORE16;
  int bf16 = 0;         // operand type: 0 fp16, 1 bf16, 2 tf32 (fp32 storage; fp32 epilogues only)
  void* out = nullptr;
  int ldo = 0;          // output leading dimension (elements)
  int grid = 0;         // persistent CTAs
  // EPI_GELU16_EXT only
  const float* xPp = nullptr;
  const float* xPm = nullptr;
  int xr = 0, xrps = 0, tpart_ld = 0;
  float* tpart = nullptr;
  // per-column bias added to the accumulator before the activation / residual (OPT
  // arch); rows >= bias_rps read bias + bias_vstride (the -eps copy under full scope)
  const float* bias = nullptr;
  int bias_rps = 0;
  long bias_vstride = 0;
  int relu = 0;  // EPI_GELU16*: ReLU instead of GELU-tanh (OPT arch)
  // EPI_UPDATE64: the fp32 master (upd_w64 cast, row stride upd_ld64) and its 16-bit shadow
  // (row stride upd_ld16); upd_transposed = 1 (required): D = V U^T, D[j, i] updates W[i, j]
  // and W16T[j, i] (projections) or W16[i, j] (upd_shadow_rm: the embedding)
  double* upd_w64 = nullptr;
  void* upd_w16 = nullptr;
  int upd_ld64 = 0, upd_ld16 = 0, upd_transposed = 0;
  int upd_m32 = 0;  // upd_w64 holds fp32 values (required: the tensor update mode's fp32 master)
  int upd_shadow_rm = 0;  // upd_transposed with a row-major shadow W16[i][j] (the embedding, fp32 master)
  int res_tma = 0;  // the output goes through tmO (set by gemm_plan): EPI_RESID32 as a
                    // cp.reduce.async.bulk add, the 16-bit epilogues as TMA stores
  const double* upd_out4 = nullptr;
  double upd_lr = 0.0, upd_scale = 1.0;
  const unsigned* upd_abort = nullptr;
  // diagnostic timeline (zo_trace_gemm): per CTA 64 globaltimer stamps -- [0] start, [1] end,
  // [2+2i, 3+2i] MMA window of segment i (i < 15), [32+2i, 33+2i] its epilogue window
  unsigned long long* trace = nullptr;
  // half-width tail: tiles [half_dp, tiles) run as two N/2-wide tiles each (half_n = 1)
  int half_dp = 0, half_n = 0;
  // split-K (gemm_enable_splitk): non-persistent, one (tile, k-chunk) per CTA, fp32 partials
  int ksplit = 0, kchunk = 0;
  long split_stride = 0;
  // stream-K split of the k-iteration space over the persistent CTAs (gemm_enable_streamk)
  int sk = 0, sk_w = 0, sk_dp = 0;
  float* sk_ws = nullptr;       // [grid][128][bn] fp32 partials of split tiles
  unsigned* sk_flags = nullptr; // [grid], zero between launches
};

// workspace needed by gemm_enable_streamk: floats / flags
inline size_t gemm_sk_ws_floats(int num_sms) { return (size_t)num_sms * 128 * 256; }
void gemm_enable_streamk(GemmDesc& g, float* ws, unsigned* flags, int num_sms);
// a mostly-empty last wave that stream-K does not take (too short a k-range per unit) runs as
// twice as many half-width tiles: the tail's MMA time and its exposed epilogue halve
void gemm_enable_halftail(GemmDesc& g, int num_sms);

// 2-D K-major tensor map over a row-major [rows, cols] matrix (row stride ld elements) of
// operand type dtype (0 fp16, 1 bf16, 2 fp32 read as tf32).
void make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                  uint32_t box_rows, int dtype);
// Fill a GemmDesc. A is [Mpad, lda] (lda >= Kp), B is [N, ldb]; dtype as make_tmap_2d.
// bn_hint: force the tile width (64 / 128 / 256) instead of the occupancy heuristic.
void gemm_plan(GemmDesc& g, const void* A, int M, int lda, const void* B, int N, int ldb, int Kp_used,
               int epi, int dtype, void* out, int ldo, int num_sms, int bn_hint = 0);
void gemm_launch(const GemmDesc& g, cudaStream_t st);
// EPI_GELU16_EXT: the number of extension-partial slots (min(bn, 128) columns each) over N
inline int gemm_ext_slots(const GemmDesc& g, int N) {
  const int s = g.bn < 128 ? g.bn : 128;
  return (N + s - 1) / s;
}
// skinny GEMMs (few output tiles, long K -- the high-rank LoRA-extension t = a . P): split K over
// `splits` CTAs per tile; partial s lands at out + s * split_stride (EPI_STORE32), summed by the
// caller in a fixed order.  Returns the number of splits used.
int gemm_enable_splitk(GemmDesc& g, int splits, long split_stride);
// EPI_UPDATE64 on a projection (upd_transposed): after gemm_plan and the upd_* fields, build the
// float64 master map the kernel streams W64 blocks through (TMA load -> update -> TMA store)
void gemm_set_update_master(GemmDesc& g);

}  // namespace zo
