// "real32" scorer support: the reference's fp32 forward (model.py:149-199 with
// _precision_dtype = float32) on the tcgen05 tensor cores by the 3xTF32 split.
//
// Every fp32 operand x is split into a tf32 "big" part b = rn_tf32(x) and the fp32
// remainder s = x - b (exact).  A K-wide product is run as ONE 3K-wide tf32 GEMM
//     [a_b | a_b | a_s] . [w_b ; w_s ; w_b]  =  a_b w_b + a_b w_s + a_s w_b,
// fp32 accumulate in TMEM: ~fp32 accuracy (the dropped a_s w_s term is ~2^-22 relative).
// The rank-r LoRA term rides in the same GEMM as 3r extra K columns
//     A: (t_b, t_b, t_s) per rank, t = a . P_s (P_s = A_win +- eps U, fp32)
//     B: (V_b, V_s, V_b) per rank
// so x . W_eff = x . W0 + (x . P_s) V^T is never materialised (adapter.py:200-234).
//
// Kernels: weight split (float64 master -> [n, 3m + ext] K-major, refreshed per scoring
// call), LN + activation split, activation split (+GELU/ReLU), fp32 causal attention.
#include <cuda_runtime.h>
#include <stdint.h>

#include "zo_common.cuh"
#include "zo_precise.h"

namespace zo {

__device__ __forceinline__ float tf32_big(float x) {
  // round-to-nearest to 10 explicit mantissa bits (the tf32 operand keeps the top 19 bits)
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) return x;  // inf / nan pass through
  u += 0x00000fffu + ((u >> 13) & 1u);
  return __uint_as_float(u & 0xffffe000u);
}

__device__ __forceinline__ float warp_sum32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum of N values per thread (blockDim.x multiple of 32, <= 1024)
template <int N>
__device__ __forceinline__ void block_sum32(float (&v)[N], float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = warp_sum32(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) red[warp * N + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) {
    float s = 0.f;
    for (int w = 0; w < nw; ++w) s += red[w * N + k];
    v[k] = s;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ weight split
// transposed (projection): W64 (in, out) [m, n] -> B'[j][i] rows j < n:
//   [0, m) w_b, [m, 2m) w_s, [2m, 3m) w_b, then per rank k: (V_b, V_s, V_b), zero pad to ldk
// not transposed (embed as the LM-head B operand): B'[v] = [E_b | E_s | E_b] of row v.
__global__ void k_split_weight_T(const double* __restrict__ W, int m, int n, float* __restrict__ out, int ldk) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int i = i0 + y, j = j0 + threadIdx.x;
    tile[y][threadIdx.x] = (i < m && j < n) ? (float)W[(size_t)i * n + j] : 0.f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int j = j0 + y, i = i0 + threadIdx.x;
    if (j < n && i < m) {
      const float x = tile[threadIdx.x][y];
      const float b = tf32_big(x);
      float* row = out + (size_t)j * ldk;
      row[i] = b;
      row[m + i] = x - b;
      row[2 * m + i] = b;
    }
  }
}

__global__ void k_split_weight_ext(const double* __restrict__ V, int n, int r, int m, float* __restrict__ out,
                                   int ldk) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float* row = out + (size_t)j * ldk;
  for (int k = 0; k < r; ++k) {
    const float x = V ? (float)V[(size_t)j * r + k] : 0.f;
    const float b = tf32_big(x);
    row[3 * m + 3 * k] = b;
    row[3 * m + 3 * k + 1] = x - b;
    row[3 * m + 3 * k + 2] = b;
  }
  for (int c = 3 * m + 3 * r; c < ldk; ++c) row[c] = 0.f;
}

__global__ void k_split_weight_rows(const double* __restrict__ W, int64_t rows, int m, float* __restrict__ out,
                                    int ldk) {
  const int64_t row = blockIdx.x;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const float x = (float)W[row * m + i];
    const float b = tf32_big(x);
    float* o = out + row * ldk;
    o[i] = b;
    o[m + i] = x - b;
    o[2 * m + i] = b;
  }
  for (int c = 3 * m + threadIdx.x; c < ldk; c += blockDim.x) out[row * ldk + c] = 0.f;
}

void launch_split_weight(const double* W64, int m, int n, const double* V, int r, float* out, int ldk,
                         int transposed, cudaStream_t st) {
  if (transposed) {
    dim3 grid((n + 31) / 32, (m + 31) / 32);
    k_split_weight_T<<<grid, dim3(32, 8), 0, st>>>(W64, m, n, out, ldk);
    k_split_weight_ext<<<(n + 255) / 256, 256, 0, st>>>(V, n, r, m, out, ldk);
  } else {
    k_split_weight_rows<<<m, 256, 0, st>>>(W64, (int64_t)m, n, out, ldk);
  }
  ZO_CUDA_TRY(cudaGetLastError());
}

// ------------------------------------------------------------------ activation split
// dst row = [a_b | a_b | a_s | (t_b, t_b, t_s) per rank | 0 pad], a = act(src row),
// t_k = sum_i a_i P[i][k] with P = Pp for rows < rps, else Pm (fp32, fixed order).
// act: 0 identity, 1 GELU-tanh (model.py:145-146, accurate tanhf), 2 ReLU (OPT).
// One CTA per row.
template <int R>
__global__ void __launch_bounds__(256) k_split_act(const float* __restrict__ src, int lds, int M, int K,
                                                   float* __restrict__ dst, int ldd, const float* __restrict__ Pp,
                                                   const float* __restrict__ Pm, int r, int rps, int act) {
  __shared__ float red[32 * (R > 0 ? R : 1)];
  const int row = blockIdx.x;
  if (row >= M) return;
  const float* s = src + (size_t)row * lds;
  float* d = dst + (size_t)row * ldd;
  const float* P = row < rps ? Pp : Pm;
  float t[R > 0 ? R : 1];
#pragma unroll
  for (int k = 0; k < (R > 0 ? R : 1); ++k) t[k] = 0.f;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    float a = s[i];
    if (act == 1) a = 0.5f * a * (1.0f + tanhf(0.7978845608028654f * (a + 0.044715f * a * a * a)));
    else if (act == 2) a = fmaxf(a, 0.f);
    const float b = tf32_big(a);
    d[i] = b;
    d[K + i] = b;
    d[2 * K + i] = a - b;
    if constexpr (R > 0) {
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k < r) t[k] += a * P[(size_t)i * r + k];
    }
  }
  int c0 = 3 * K;
  if constexpr (R > 0) {
    block_sum32<R>(t, red);
    if (threadIdx.x == 0)
      for (int k = 0; k < r && k < R; ++k) {
        const float b = tf32_big(t[k]);
        d[3 * K + 3 * k] = b;
        d[3 * K + 3 * k + 1] = b;
        d[3 * K + 3 * k + 2] = t[k] - b;
      }
    c0 = 3 * K + 3 * r;
  }
  for (int c = c0 + threadIdx.x; c < ldd; c += blockDim.x) d[c] = 0.f;
}

// LN (model.py:139-142, eps 1e-5) then the activation split of k_split_act.
// Rows >= rps read gamma/beta + vstride (full scope: the -eps copy).
template <int R>
__global__ void __launch_bounds__(256) k_ln_split(const float* __restrict__ x32, const float* __restrict__ g,
                                                  const float* __restrict__ bta, long vstride, int M, int d,
                                                  float* __restrict__ dst, int ldd, const float* __restrict__ Pp,
                                                  const float* __restrict__ Pm, int r, int rps) {
  __shared__ float red[32 * (R > 1 ? R : 2)];
  const int row = blockIdx.x;
  if (row >= M) return;
  const float* x = x32 + (size_t)row * d;
  float* o = dst + (size_t)row * ldd;
  const long vo = row < rps ? 0 : vstride;
  const float* P = row < rps ? Pp : Pm;
  float s1[1] = {0.f};
  for (int i = threadIdx.x; i < d; i += blockDim.x) s1[0] += x[i];
  block_sum32<1>(s1, red);
  const float mu = s1[0] / (float)d;
  float s2[1] = {0.f};
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float c = x[i] - mu;
    s2[0] += c * c;
  }
  block_sum32<1>(s2, red);
  const float rstd = 1.0f / sqrtf(s2[0] / (float)d + 1e-5f);
  float t[R > 0 ? R : 1];
#pragma unroll
  for (int k = 0; k < (R > 0 ? R : 1); ++k) t[k] = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float h = (x[i] - mu) * rstd * g[vo + i] + bta[vo + i];
    const float b = tf32_big(h);
    o[i] = b;
    o[d + i] = b;
    o[2 * d + i] = h - b;
    if constexpr (R > 0) {
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k < r) t[k] += h * P[(size_t)i * r + k];
    }
  }
  int c0 = 3 * d;
  if constexpr (R > 0) {
    block_sum32<R>(t, red);
    if (threadIdx.x == 0)
      for (int k = 0; k < r && k < R; ++k) {
        const float b = tf32_big(t[k]);
        o[3 * d + 3 * k] = b;
        o[3 * d + 3 * k + 1] = b;
        o[3 * d + 3 * k + 2] = t[k] - b;
      }
    c0 = 3 * d + 3 * r;
  }
  for (int c = c0 + threadIdx.x; c < ldd; c += blockDim.x) o[c] = 0.f;
}

#define ZO_RANK_DISPATCH(KERNEL, ...)                                  \
  do {                                                                 \
    if (r <= 0) KERNEL<0><<<M, 256, 0, st>>>(__VA_ARGS__);             \
    else if (r <= 2) KERNEL<2><<<M, 256, 0, st>>>(__VA_ARGS__);        \
    else if (r <= 4) KERNEL<4><<<M, 256, 0, st>>>(__VA_ARGS__);        \
    else KERNEL<8><<<M, 256, 0, st>>>(__VA_ARGS__);                    \
  } while (0)

void launch_split_act(const float* src, int lds, int M, int K, float* dst, int ldd, const float* Pp,
                      const float* Pm, int r, int rps, int act, cudaStream_t st) {
  if (r > 8) throw Error(ZO_ERR_CONFIG, "real32 scorer supports rank <= 8");
  ZO_RANK_DISPATCH(k_split_act, src, lds, M, K, dst, ldd, Pp, Pm, r, rps, act);
  ZO_CUDA_TRY(cudaGetLastError());
}

void launch_ln_split(const float* x32, const float* gamma, const float* beta, long vstride, int M, int d,
                     float* dst, int ldd, const float* Pp, const float* Pm, int r, int rps, cudaStream_t st) {
  if (r > 8) throw Error(ZO_ERR_CONFIG, "real32 scorer supports rank <= 8");
  ZO_RANK_DISPATCH(k_ln_split, x32, gamma, beta, vstride, M, d, dst, ldd, Pp, Pm, r, rps);
  ZO_CUDA_TRY(cudaGetLastError());
}

// ------------------------------------------------------------------ fp32 causal attention
// model.py:184-194 in fp32: s = q k^T / sqrt(dh), causal mask, s - max, exp, / sum, a v.
// One CTA (4 warps) per (sequence, head); K and V of the head staged in shared memory in
// chunks of 64 keys; a warp owns query rows w, w+4, ...  qkv row layout [q | k | v], d each.
__global__ void __launch_bounds__(128) k_attn32(const float* __restrict__ qkv, int ldq, float* __restrict__ ctx,
                                                int ldc, int T, int H, int dh) {
  extern __shared__ float sm[];
  const int seq = blockIdx.x / H, h = blockIdx.x % H;
  const int d = H * dh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Ks = sm;                 // [64][dh + 1]
  float* Vs = sm + 64 * (dh + 1);  // [64][dh]
  float* Pw = Vs + 64 * dh;        // per warp [64] probabilities of the current chunk
  float* Qw = Pw + 4 * 64;         // per warp [dh] query row
  const float scale = 1.0f / sqrtf((float)dh);
  const float* base = qkv + (size_t)seq * T * ldq;
  // per query row state kept by its warp: running max, sum, output (dh / 32 values per lane)
  const int nq = (T + 3) / 4;
  for (int qi = 0; qi < nq; ++qi) {
    const int t = qi * 4 + warp;  // this warp's query row
    float m = -INFINITY, l = 0.f;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};  // dh <= 128
    if (t < T)
      for (int c = lane; c < dh; c += 32) Qw[warp * dh + c] = base[(size_t)t * ldq + h * dh + c];
    // every warp walks the key chunks up to the block's last query row of this round
    const int tmax = min(T - 1, qi * 4 + 3);
    for (int j0 = 0; j0 <= tmax; j0 += 64) {
      const int nj = min(64, tmax + 1 - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < nj * dh; e += blockDim.x) {
        const int j = e / dh, c = e % dh;
        Ks[j * (dh + 1) + c] = base[(size_t)(j0 + j) * ldq + d + h * dh + c];
        Vs[j * dh + c] = base[(size_t)(j0 + j) * ldq + 2 * d + h * dh + c];
      }
      __syncthreads();
      if (t >= T) continue;
      // scores of keys j0 + lane, j0 + lane + 32 (causal: key <= t)
      float sc[2];
      float cm = -INFINITY;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = lane + 32 * u;
        sc[u] = -INFINITY;
        if (j < nj && j0 + j <= t) {
          float s = 0.f;
          for (int c = 0; c < dh; ++c) s += Qw[warp * dh + c] * Ks[j * (dh + 1) + c];
          sc[u] = s * scale;
        }
        cm = fmaxf(cm, sc[u]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
      if (cm == -INFINITY) continue;  // no visible key in this chunk
      const float mn = fmaxf(m, cm);
      const float corr = (m == -INFINITY) ? 0.f : expf(m - mn);
      float ps = 0.f;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = lane + 32 * u;
        const float pj = (sc[u] == -INFINITY) ? 0.f : expf(sc[u] - mn);
        if (j < 64) Pw[warp * 64 + j] = pj;
        ps += pj;
      }
      ps = warp_sum32(ps);
      l = l * corr + ps;
      m = mn;
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = lane + 32 * u;
        if (c < dh) {
          float a = acc[u] * corr;
          for (int j = 0; j < nj; ++j) a += Pw[warp * 64 + j] * Vs[j * dh + c];
          acc[u] = a;
        }
      }
      __syncwarp();
    }
    if (t < T) {
      float* o = ctx + ((size_t)seq * T + t) * ldc + h * dh;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = lane + 32 * u;
        if (c < dh) o[c] = acc[u] / l;
      }
    }
  }
}

void launch_attn32(const float* qkv, int ldq, float* ctx, int ldc, int nseq, int T, int H, int dh, cudaStream_t st) {
  if (dh > 128) throw Error(ZO_ERR_CONFIG, "real32 attention supports head dim <= 128");
  const size_t smem = (size_t)(64 * (dh + 1) + 64 * dh + 4 * 64 + 4 * dh) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    ZO_CUDA_TRY(cudaFuncSetAttribute(k_attn32, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    attr = true;
  }
  k_attn32<<<nseq * H, 128, smem, st>>>(qkv, ldq, ctx, ldc, T, H, dh);
  ZO_CUDA_TRY(cudaGetLastError());
}

}  // namespace zo
