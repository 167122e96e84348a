// "real32" scorer: the reference's fp32 forward on tcgen05 via the 3xTF32 split (precise.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace zo {

// B' operand of one matrix from its float64 master.  transposed = 1 (projection, W64 (in, out)
// [m, n]): B'[n, ldk] = [w_b | w_s | w_b | (V_b, V_s, V_b) per rank | 0]; transposed = 0
// (embed as LM-head operand, rows = vocab): B'[m, ldk] = [E_b | E_s | E_b | 0] with K = n.
void launch_split_weight(const double* W64, int m, int n, const double* V, int r, float* out, int ldk,
                         int transposed, cudaStream_t st);
// A' operand: dst[row] = [a_b | a_b | a_s | (t_b, t_b, t_s) per rank | 0], a = act(src[row, :K]),
// t = a . P_s (P_s = Pp for rows < rps, else Pm; r = 0: no extension); act 0 id, 1 GELU, 2 ReLU
void launch_split_act(const float* src, int lds, int M, int K, float* dst, int ldd, const float* Pp,
                      const float* Pm, int r, int rps, int act, cudaStream_t st);
// LN (model.py:139-142) then the A' split of launch_split_act
void launch_ln_split(const float* x32, const float* gamma, const float* beta, long vstride, int M, int d,
                     float* dst, int ldd, const float* Pp, const float* Pm, int r, int rps, cudaStream_t st);
// fp32 causal attention (model.py:184-194): qkv [nseq * T, ldq] -> ctx [nseq * T, ldc]
void launch_attn32(const float* qkv, int ldq, float* ctx, int ldc, int nseq, int T, int H, int dh, cudaStream_t st);

}  // namespace zo
