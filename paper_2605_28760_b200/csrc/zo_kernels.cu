// Scorer glue, loss extraction, coefficient, update and fold kernels.
// Reference citations are to /root/reference/pkg/src/zoserve.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "zo_common.cuh"
#include "zo_kernels.h"

namespace zo {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ float ld16(const void* p, size_t i, bool bf16) {
  const uint16_t raw = reinterpret_cast<const uint16_t*>(p)[i];
  if (bf16) return __bfloat162float(__ushort_as_bfloat16(raw));
  return __half2float(__ushort_as_half(raw));
}
__device__ __forceinline__ uint16_t to16(float v, bool bf16) {
  if (bf16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
  return __half_as_ushort(__float2half_rn(v));
}
__device__ __forceinline__ float from16(uint16_t raw, bool bf16) {
  if (bf16) return __bfloat162float(__ushort_as_bfloat16(raw));
  return __half2float(__ushort_as_half(raw));
}
__device__ __forceinline__ void st16(void* p, size_t i, float v, bool bf16) {
  reinterpret_cast<uint16_t*>(p)[i] = to16(v, bf16);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int N>
__device__ __forceinline__ void block_sum(float (&v)[N], float* red /* >= 32*N */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
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

__device__ __forceinline__ float block_max(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float m = -CUDART_INF_F;
  for (int w = 0; w < nw; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  return m;
}

// Write the LoRA extension columns for one row: t_k -> (hi, lo, hi) or t.
__device__ __forceinline__ void write_ext(void* out, size_t base, int k, float t, int ext_terms, bool bf16) {
  if (ext_terms == 3) {
    const uint16_t hi = to16(t, bf16);
    const float lo = t - from16(hi, bf16);
    uint16_t* o = reinterpret_cast<uint16_t*>(out) + base + 3 * k;
    o[0] = hi;
    o[1] = to16(lo, bf16);
    o[2] = hi;
  } else {
    reinterpret_cast<uint16_t*>(out)[base + k] = to16(t, bf16);
  }
}

// ------------------------------------------------------------------ fused-extension finalize
// t[row, k] = sum over tiles j of tpart[j][row][k].  A CTA of 256 threads owns PAIRS
// consecutive (row, k) pairs x GROUPS tile groups: group g sums tiles g, g+GROUPS, ... in
// ascending order (for a fixed tile the pairs are contiguous: coalesced), then the group
// sums are added in group order.  GROUPS is chosen from the tile count alone (8 up to 16
// tiles -- the high-rank split-K partials --, 32 above -- the fused GELU-epilogue / attention
// partials), so the summation order depends on neither M nor the launch shape.
template <int GROUPS>
__global__ void __launch_bounds__(256) k_ext_finalize(const float* __restrict__ tpart, int ntiles, int ld, int M,
                                                      int r, void* __restrict__ a, int lda, int K, int ext_terms,
                                                      bool bf16, int neg_from) {
  constexpr int PAIRS = 256 / GROUPS;
  pdl_launch_dependents();
  pdl_wait();
  __shared__ float part[GROUPS][PAIRS];
  const int p = threadIdx.x % PAIRS, g = threadIdx.x / PAIRS;
  const int64_t i = (int64_t)blockIdx.x * PAIRS + p;  // = row * r + k
  const bool ok = i < (int64_t)M * r;
  float t = 0.f;
  if (ok) {
    const float* src = tpart + i;
    const size_t stride = (size_t)ld * r;
#pragma unroll 4
    for (int j = g; j < ntiles; j += GROUPS) t += src[(size_t)j * stride];
  }
  part[g][p] = t;
  __syncthreads();
  if (g == 0 && ok) {
    float s = part[0][p];
#pragma unroll
    for (int q = 1; q < GROUPS; ++q) s += part[q][p];
    const int row = (int)(i / r), k = (int)(i % r);
    if (neg_from >= 0 && row >= neg_from) s = -s;
    write_ext(a, (size_t)row * lda + K, k, s, ext_terms, bf16);
  }
}

// few tiles (the high-rank split-K partials): a thread per (row, k) pair sums its <= 16
// partials in tile order (independent loads, unrolled) -- the grouped kernel's 32-pair CTAs
// were thousands of tiny CTAs at M x r = 2016 x 128
__global__ void __launch_bounds__(256) k_ext_finalize_flat(const float* __restrict__ tpart, int ntiles, int ld,
                                                           int M, int r, void* __restrict__ a, int lda, int K,
                                                           int ext_terms, bool bf16, int neg_from) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // = row * r + k
  if (i >= (int64_t)M * r) return;
  const float* src = tpart + i;
  const size_t stride = (size_t)ld * r;
  float t = 0.f;
#pragma unroll 4
  for (int j = 0; j < ntiles; ++j) t += src[(size_t)j * stride];
  const int row = (int)(i / r), k = (int)(i % r);
  if (neg_from >= 0 && row >= neg_from) t = -t;
  write_ext(a, (size_t)row * lda + K, k, t, ext_terms, bf16);
}

void launch_ext_finalize(const float* tpart, int ntiles, int ld, int M, int r, void* a, int lda, int K,
                         int ext_terms, bool bf16, cudaStream_t st, int neg_from) {
  const int64_t pairs = (int64_t)M * r;
  if (ntiles <= 16 && pairs >= 148 * 256)  // the high-rank split-K partials
    launch_pdl(k_ext_finalize_flat, dim3((unsigned)((pairs + 255) / 256)), dim3(256), 0, st, tpart, ntiles, ld, M,
               r, a, lda, K, ext_terms, bf16, neg_from);
  else if (ntiles <= 16)
    launch_pdl(k_ext_finalize<8>, dim3((unsigned)((pairs + 31) / 32)), dim3(256), 0, st, tpart, ntiles, ld, M, r, a,
               lda, K, ext_terms, bf16, neg_from);
  else
    launch_pdl(k_ext_finalize<32>, dim3((unsigned)((pairs + 7) / 8)), dim3(256), 0, st, tpart, ntiles, ld, M, r, a,
               lda, K, ext_terms, bf16, neg_from);
}

// ------------------------------------------------------------------ embed
__global__ void k_embed(float* __restrict__ x32, const int32_t* __restrict__ tokens, int tok_ld, int B, int T, int d,
                        const double* __restrict__ E64, const float* __restrict__ E32,
                        const void* __restrict__ E16, bool bf16, const float* __restrict__ Pp, const float* __restrict__ Pm, const float* __restrict__ Ve,
                        int r, const float* __restrict__ pe, PosEmbed pos) {
  const int row = blockIdx.x;
  const int per_sign = B * T;
  const int s = row / per_sign, rem = row % per_sign, b = rem / T, t = rem % T;
  const int tok = tokens[b * tok_ld + t];
  const float* P = (s == 0 ? Pp : Pm) + (size_t)tok * r;
  const size_t prow = (size_t)(t + pos.offset);
  const float* PP = pos.W64 ? (s == 0 ? pos.Pp : pos.Pm) + prow * r : nullptr;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float e = E64 ? (float)E64[(size_t)tok * d + i] : E32 ? E32[(size_t)tok * d + i] : ld16(E16, (size_t)tok * d + i, bf16);
    float delta = 0.f;
    for (int k = 0; k < r; ++k) delta += P[k] * Ve[(size_t)i * r + k];
    float pv;
    if (PP) {  // OPT: inputs_embeds + embed_positions(t + 2), each with its LoRA delta
      float pd = 0.f;
      for (int k = 0; k < r; ++k) pd += PP[k] * pos.V32[(size_t)i * r + k];
      pv = (float)pos.W64[prow * d + i] + pd;
    } else {
      pv = pe[(size_t)t * d + i];
    }
    x32[(size_t)row * d + i] = (e + delta) + pv;
  }
}

// High rank (r % 32 == 0): the delta P_s[tok] . V_e^T is a [rows x r] x [r x d] product --
// a CTA computes 32 rows x 128 columns with 32-wide rank slices of P and V staged in
// shared memory (V transposed, padded against bank conflicts), k ascending per element as
// in k_embed.  The learned-position (OPT) form keeps k_embed.
constexpr int EHR_ROWS = 32, EHR_COLS = 128, EHR_K = 32;
__global__ void __launch_bounds__(EHR_COLS) k_embed_hr(float* __restrict__ x32, const int32_t* __restrict__ tokens,
                                                       int tok_ld, int B, int T, int d,
                                                       const double* __restrict__ E64, const float* __restrict__ E32,
                                                       const void* __restrict__ E16, bool bf16,
                                                       const float* __restrict__ Pp,
                                                       const float* __restrict__ Pm, const float* __restrict__ Ve,
                                                       int r, const float* __restrict__ pe, int nrows) {
  __shared__ float Ps[EHR_ROWS][EHR_K];
  __shared__ float Vs[EHR_K][EHR_COLS + 1];
  __shared__ int toks[EHR_ROWS];
  const int i = blockIdx.x * EHR_COLS + threadIdx.x;
  const int row0 = blockIdx.y * EHR_ROWS;
  const int per_sign = B * T;
  if (threadIdx.x < EHR_ROWS) {
    const int row = row0 + threadIdx.x;
    int tk = 0;
    if (row < nrows) {
      const int rem = row % per_sign;
      tk = tokens[(rem / T) * tok_ld + rem % T];
    }
    toks[threadIdx.x] = tk;
  }
  float acc[EHR_ROWS];
#pragma unroll
  for (int q = 0; q < EHR_ROWS; ++q) acc[q] = 0.f;
  __syncthreads();
  for (int k0 = 0; k0 < r; k0 += EHR_K) {
    for (int e = threadIdx.x; e < EHR_ROWS * EHR_K; e += EHR_COLS) {
      const int rr = e / EHR_K, kk = e % EHR_K, row = row0 + rr;
      const float* P = (row < per_sign) ? Pp : Pm;
      Ps[rr][kk] = row < nrows ? P[(size_t)toks[rr] * r + k0 + kk] : 0.f;
    }
    for (int e = threadIdx.x; e < EHR_COLS * EHR_K; e += EHR_COLS) {
      const int c = e / EHR_K, kk = e % EHR_K, col = blockIdx.x * EHR_COLS + c;
      Vs[kk][c] = col < d ? Ve[(size_t)col * r + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < EHR_K; ++kk) {
      const float v = Vs[kk][threadIdx.x];
#pragma unroll
      for (int q = 0; q < EHR_ROWS; ++q) acc[q] += Ps[q][kk] * v;
    }
    __syncthreads();
  }
  if (i >= d) return;
#pragma unroll
  for (int q = 0; q < EHR_ROWS; ++q) {
    const int row = row0 + q;
    if (row >= nrows) break;
    const int t = (row % per_sign) % T, tk = toks[q];
    const float e = E64 ? (float)E64[(size_t)tk * d + i] : E32 ? E32[(size_t)tk * d + i] : ld16(E16, (size_t)tk * d + i, bf16);
    x32[(size_t)row * d + i] = (e + acc[q]) + pe[(size_t)t * d + i];
  }
}

void launch_embed(float* x32, const int32_t* tokens, int tok_ld, int B, int T, int d, const double* E64,
                  const float* E32, const void* E16, bool bf16, const float* Pplus, const float* Pminus, const float* Ve32, int r,
                  const float* pe, const PosEmbed& pos, int nrows, cudaStream_t st) {
  if (r > 8 && r % EHR_K == 0 && !pos.W64) {
    const dim3 grid((unsigned)ceil_div(d, EHR_COLS), (unsigned)ceil_div(nrows, EHR_ROWS));
    k_embed_hr<<<grid, EHR_COLS, 0, st>>>(x32, tokens, tok_ld, B, T, d, E64, E32, E16, bf16, Pplus, Pminus, Ve32, r, pe,
                                          nrows);
    return;
  }
  k_embed<<<nrows, 256, 0, st>>>(x32, tokens, tok_ld, B, T, d, E64, E32, E16, bf16, Pplus, Pminus, Ve32, r, pe, pos);
}

// ------------------------------------------------------------------ LN (+ extension), warp per row

__device__ __forceinline__ void store4_16(void* out, size_t i, float a, float b, float c, float d, bool bf16) {
  uint2 w;
  w.x = (uint32_t)to16(a, bf16) | ((uint32_t)to16(b, bf16) << 16);
  w.y = (uint32_t)to16(c, bf16) | ((uint32_t)to16(d, bf16) << 16);
  *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(out) + i) = w;
}

// h = LN(x) -> out[:, :d] (16-bit), ext columns t = h . P_s (fp32 h), one warp per row,
// float4 loads (the row stays in L1 across the three passes).
__global__ void __launch_bounds__(256) k_ln_ext(const float* __restrict__ x32, const float* __restrict__ g,
                                                const float* __restrict__ bta, int M, int d, void* __restrict__ out,
                                                int ldo, bool bf16, const float* __restrict__ Pp,
                                                const float* __restrict__ Pm, int r, int rows_per_sign,
                                                int ext_terms, long vstride) {
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float4* x = reinterpret_cast<const float4*>(x32 + (size_t)row * d);
  const int n4 = d >> 2;
  float s = 0.f;
#pragma unroll 4
  for (int i = lane; i < n4; i += 32) {
    const float4 v = x[i];
    s += (v.x + v.y) + (v.z + v.w);
  }
  const float mu = warp_sum(s) / (float)d;
  s = 0.f;
#pragma unroll 4
  for (int i = lane; i < n4; i += 32) {
    const float4 v = x[i];
    const float a = v.x - mu, b = v.y - mu, c = v.z - mu, e = v.w - mu;
    s += (a * a + b * b) + (c * c + e * e);
  }
  const float rsd = 1.0f / sqrtf(warp_sum(s) / (float)d + 1e-5f);
  const float* P = (row < rows_per_sign) ? Pp : Pm;
  // full scope: the -eps probe rows read the second (VectorProbe -1) copy of the LN params
  const long voff = (row < rows_per_sign) ? 0 : vstride;
  const float4* g4 = reinterpret_cast<const float4*>(g + voff);
  const float4* b4 = reinterpret_cast<const float4*>(bta + voff);
  for (int k0 = 0; k0 < (r > 0 ? r : 1); k0 += 8) {
    float t[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int kn = min(8, r - k0);
    for (int i = lane; i < n4; i += 32) {
      const float4 v = x[i], gg = g4[i], bb = b4[i];
      float h[4] = {(v.x - mu) * rsd * gg.x + bb.x, (v.y - mu) * rsd * gg.y + bb.y,
                    (v.z - mu) * rsd * gg.z + bb.z, (v.w - mu) * rsd * gg.w + bb.w};
      if (k0 == 0) store4_16(out, (size_t)row * ldo + 4 * i, h[0], h[1], h[2], h[3], bf16);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float* pr = P + (size_t)(4 * i + e) * r + k0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < kn) t[q] += h[e] * pr[q];
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = warp_sum(t[q]);
    if (lane == 0)
      for (int q = 0; q < kn; ++q) write_ext(out, (size_t)row * ldo + d, k0 + q, t[q], ext_terms, bf16);
  }
}

// Register-resident variant: the whole row (NV float4 per lane) is loaded once
// with NV independent 16-byte loads in flight per lane, then mean, variance
// (two-pass, in registers), h and the extension dots.  One HBM read of x.
template <int NV, int XR>
__global__ void __launch_bounds__(256) k_ln_ext_reg(const float* __restrict__ x32, const float* __restrict__ g,
                                                    const float* __restrict__ bta, int M, void* __restrict__ out,
                                                    int ldo, bool bf16, const float* __restrict__ Pp,
                                                    const float* __restrict__ Pm, int rows_per_sign,
                                                    int ext_terms, long vstride) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int d = NV * 128;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float4* x = reinterpret_cast<const float4*>(x32 + (size_t)row * d);
  float4 v[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = x[lane + 32 * j];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
  const float mu = warp_sum(s) / (float)d;
  s = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const float a = v[j].x - mu, b = v[j].y - mu, c = v[j].z - mu, e = v[j].w - mu;
    s += (a * a + b * b) + (c * c + e * e);
  }
  const float rsd = 1.0f / sqrtf(warp_sum(s) / (float)d + 1e-5f);
  const float* P = (row < rows_per_sign) ? Pp : Pm;
  // full scope: the -eps probe rows read the second (VectorProbe -1) copy of the LN params
  const long voff = (row < rows_per_sign) ? 0 : vstride;
  const float4* g4 = reinterpret_cast<const float4*>(g + voff);
  const float4* b4 = reinterpret_cast<const float4*>(bta + voff);
  float t[XR > 0 ? XR : 1];
#pragma unroll
  for (int k = 0; k < (XR > 0 ? XR : 1); ++k) t[k] = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i = lane + 32 * j;
    const float4 gg = g4[i], bb = b4[i];
    const float h[4] = {(v[j].x - mu) * rsd * gg.x + bb.x, (v[j].y - mu) * rsd * gg.y + bb.y,
                        (v[j].z - mu) * rsd * gg.z + bb.z, (v[j].w - mu) * rsd * gg.w + bb.w};
    store4_16(out, (size_t)row * ldo + 4 * i, h[0], h[1], h[2], h[3], bf16);
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int k = 0; k < XR; ++k) t[k] += h[e] * P[(size_t)(4 * i + e) * XR + k];
  }
#pragma unroll
  for (int k = 0; k < XR; ++k) t[k] = warp_sum(t[k]);
  if (lane == 0)
    for (int k = 0; k < XR; ++k) write_ext(out, (size_t)row * ldo + d, k, t[k], ext_terms, bf16);
}

// CTA per R rows (R = 2 when the rows pair up within one probe sign), 256 threads,
// NPT float4 per thread and row in registers: one HBM read of x, and the LN
// parameters / probe operand P (2 + r floats per column, the larger share of the
// bytes a row touches) are loaded once for the R rows, which also share each
// block-reduction round.
template <int NPT, int XR, int R>
__global__ void __launch_bounds__(256, NPT <= 5 ? 4 : 2) k_ln_row(const float* __restrict__ x32, const float* __restrict__ g,
                                                const float* __restrict__ bta, int d, void* __restrict__ out, int ldo,
                                                bool bf16, const float* __restrict__ Pp, const float* __restrict__ Pm,
                                                int rows_per_sign, int ext_terms, long vstride) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ float red[8 * R * (XR + 1)];
  const int row0 = blockIdx.x * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  float4 v[R][NPT];
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    const float4* x = reinterpret_cast<const float4*>(x32 + (size_t)(row0 + rr) * d);
#pragma unroll
    for (int j = 0; j < NPT; ++j) v[rr][j] = x[tid + j * blockDim.x];
  }
  // block sums of R values per round, fixed order
  auto bsum = [&](float (&a)[R]) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) a[rr] = warp_sum(a[rr]);
    __syncthreads();  // the previous round's reads of red[] are done
    if (lane == 0)
#pragma unroll
      for (int rr = 0; rr < R; ++rr) red[warp * R + rr] = a[rr];
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      float tot = 0.f;
      for (int w = 0; w < nw; ++w) tot += red[w * R + rr];
      a[rr] = tot;
    }
  };
  float mu[R], rsd[R];
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NPT; ++j) s += (v[rr][j].x + v[rr][j].y) + (v[rr][j].z + v[rr][j].w);
    mu[rr] = s;
  }
  bsum(mu);
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    mu[rr] = mu[rr] / (float)d;
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const float a = v[rr][j].x - mu[rr], b = v[rr][j].y - mu[rr], c = v[rr][j].z - mu[rr], e = v[rr][j].w - mu[rr];
      s += (a * a + b * b) + (c * c + e * e);
    }
    rsd[rr] = s;
  }
  bsum(rsd);
#pragma unroll
  for (int rr = 0; rr < R; ++rr) rsd[rr] = 1.0f / sqrtf(rsd[rr] / (float)d + 1e-5f);
  const bool plus = row0 < rows_per_sign;  // the R rows share one probe sign
  const float* P = plus ? Pp : Pm;
  // full scope: the -eps probe rows read the second (VectorProbe -1) copy of the LN params
  const long voff = plus ? 0 : vstride;
  const float4* g4 = reinterpret_cast<const float4*>(g + voff);
  const float4* b4 = reinterpret_cast<const float4*>(bta + voff);
  float t[R][XR > 0 ? XR : 1];
#pragma unroll
  for (int rr = 0; rr < R; ++rr)
#pragma unroll
    for (int k = 0; k < XR; ++k) t[rr][k] = 0.f;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int i = tid + j * blockDim.x;
    const float4 gg = g4[i], bb = b4[i];
    float4 p01 = make_float4(0.f, 0.f, 0.f, 0.f), p23 = p01;
    if constexpr (XR == 2) {
      const float4* pr = reinterpret_cast<const float4*>(P + (size_t)(4 * i) * 2);
      p01 = pr[0];  // P[4i..4i+1][0..1]
      p23 = pr[1];  // P[4i+2..4i+3][0..1]
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const float h[4] = {(v[rr][j].x - mu[rr]) * rsd[rr] * gg.x + bb.x, (v[rr][j].y - mu[rr]) * rsd[rr] * gg.y + bb.y,
                          (v[rr][j].z - mu[rr]) * rsd[rr] * gg.z + bb.z, (v[rr][j].w - mu[rr]) * rsd[rr] * gg.w + bb.w};
      store4_16(out, (size_t)(row0 + rr) * ldo + 4 * i, h[0], h[1], h[2], h[3], bf16);
      if constexpr (XR == 2) {
        t[rr][0] += h[0] * p01.x + h[1] * p01.z + h[2] * p23.x + h[3] * p23.z;
        t[rr][1] += h[0] * p01.y + h[1] * p01.w + h[2] * p23.y + h[3] * p23.w;
      } else if constexpr (XR > 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int k = 0; k < XR; ++k) t[rr][k] += h[e] * P[(size_t)(4 * i + e) * XR + k];
      }
    }
  }
  if constexpr (XR == 0) return;
#pragma unroll
  for (int rr = 0; rr < R; ++rr)
#pragma unroll
    for (int k = 0; k < XR; ++k) t[rr][k] = warp_sum(t[rr][k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int k = 0; k < XR; ++k) red[8 * R + (warp * R + rr) * XR + k] = t[rr][k];
  __syncthreads();
  if (tid < R * XR) {
    const int rr = tid / XR, k = tid % XR;
    float a = 0.f;
    for (int w = 0; w < nw; ++w) a += red[8 * R + (w * R + rr) * XR + k];
    write_ext(out, (size_t)(row0 + rr) * ldo + d, k, a, ext_terms, bf16);
  }
}

template <int NPT>
static bool ln_row_dispatch(const float* x32, const float* gamma, const float* beta, int M, int d, void* out, int ldo,
                            bool bf16, const float* Pp, const float* Pm, int r, int rps, int ext_terms, long vstride,
                            cudaStream_t st) {
  const int threads = d / (4 * NPT);
  if (threads * 4 * NPT != d || threads % 32 || threads > 256) return false;
  const bool pair = (M % 2 == 0) && (rps % 2 == 0);  // row pairs never straddle the probe signs
#define ZO_LNR(XR)                                                                                              \
  case XR:                                                                                                      \
    if (pair)                                                                                                   \
      launch_pdl(k_ln_row<NPT, XR, 2>, dim3(M / 2), dim3(threads), 0, st, x32, gamma, beta, d, out, ldo, bf16, \
                 Pp, Pm, rps, ext_terms, vstride);                                                              \
    else                                                                                                        \
      launch_pdl(k_ln_row<NPT, XR, 1>, dim3(M), dim3(threads), 0, st, x32, gamma, beta, d, out, ldo, bf16, Pp, \
                 Pm, rps, ext_terms, vstride);                                                                  \
    return true;
  switch (r) {
    ZO_LNR(0)
    ZO_LNR(1)
    ZO_LNR(2)
    ZO_LNR(4)
    default: return false;
  }
#undef ZO_LNR
}

template <int NV>
static bool ln_reg_dispatch(const float* x32, const float* gamma, const float* beta, int M, void* out, int ldo,
                            bool bf16, const float* Pp, const float* Pm, int r, int rps, int ext_terms, long vstride,
                            cudaStream_t st) {
  const int grid = (M + 7) / 8;
  switch (r) {
    case 1: launch_pdl(k_ln_ext_reg<NV, 1>, dim3(grid), dim3(256), 0, st, x32, gamma, beta, M, out, ldo, bf16, Pp, Pm, rps, ext_terms, vstride); return true;
    case 2: launch_pdl(k_ln_ext_reg<NV, 2>, dim3(grid), dim3(256), 0, st, x32, gamma, beta, M, out, ldo, bf16, Pp, Pm, rps, ext_terms, vstride); return true;
    case 4: launch_pdl(k_ln_ext_reg<NV, 4>, dim3(grid), dim3(256), 0, st, x32, gamma, beta, M, out, ldo, bf16, Pp, Pm, rps, ext_terms, vstride); return true;
    default: return false;
  }
}

void launch_ln_ext(const float* x32, const float* gamma, const float* beta, int M, int d, void* out, int ldo,
                   bool bf16, const float* Pplus, const float* Pminus, int r, int rows_per_sign, int ext_terms,
                   long vstride, cudaStream_t st) {
  if (d % 4 || ldo % 4) throw Error(ZO_ERR_DIMENSION, "LN rows must be multiples of 4");
  bool done = false;
  // CTA-per-row kernel (d multiple of 128 and <= 8192); measured against the warp-per-row
  // register kernel at d = 5120: 20.1 vs 36.7 us
  if (d % 1024 == 0) {
    switch (d / 1024) {
      case 1: done = ln_row_dispatch<1>(x32, gamma, beta, M, d, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
      case 2: done = ln_row_dispatch<2>(x32, gamma, beta, M, d, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
      case 4: done = ln_row_dispatch<4>(x32, gamma, beta, M, d, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
      case 5: done = ln_row_dispatch<5>(x32, gamma, beta, M, d, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
      case 8: done = ln_row_dispatch<8>(x32, gamma, beta, M, d, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
      default: break;
    }
  } else if (d % 128 == 0 && d <= 1024) {
    done = ln_row_dispatch<1>(x32, gamma, beta, M, d, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms,
                              vstride, st);
  }
  if (!done) switch (d) {
    case 768: done = ln_reg_dispatch<6>(x32, gamma, beta, M, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
    case 1024: done = ln_reg_dispatch<8>(x32, gamma, beta, M, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
    case 2048: done = ln_reg_dispatch<16>(x32, gamma, beta, M, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
    case 4096: done = ln_reg_dispatch<32>(x32, gamma, beta, M, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
    case 5120: done = ln_reg_dispatch<40>(x32, gamma, beta, M, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms, vstride, st); break;
    default: break;
  }
  if (!done)
    launch_pdl(k_ln_ext, dim3((M + 7) / 8), dim3(256), 0, st, x32, gamma, beta, M, d, out, ldo, bf16, Pplus, Pminus, r, rows_per_sign,
                                          ext_terms, vstride);
}

// ------------------------------------------------------------------ extension of a 16-bit activation
// t_k = a[row, :K] . P_s[:, k] -> ext columns, one warp per row, 16-byte loads.
__global__ void __launch_bounds__(256) k_ext(void* __restrict__ a, int lda, int M, int K, bool bf16,
                                             const float* __restrict__ Pp, const float* __restrict__ Pm, int r,
                                             int rows_per_sign, int ext_terms) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float* P = (row < rows_per_sign) ? Pp : Pm;
  const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a) + (size_t)row * lda);
  const int n8 = K >> 3;
  for (int k0 = 0; k0 < r; k0 += 8) {
    float t[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int kn = min(8, r - k0);
    for (int i = lane; i < n8; i += 32) {
      const uint4 w = src[i];
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v = from16((uint16_t)(ww[e >> 1] >> (16 * (e & 1))), bf16);
        const float* pr = P + (size_t)(8 * i + e) * r + k0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < kn) t[q] += v * pr[q];
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = warp_sum(t[q]);
    if (lane == 0)
      for (int q = 0; q < kn; ++q) write_ext(a, (size_t)row * lda + K, k0 + q, t[q], ext_terms, bf16);
  }
}

void launch_ext(void* a, int lda, int M, int K, bool bf16, const float* Pplus, const float* Pminus, int r,
                int rows_per_sign, int ext_terms, cudaStream_t st) {
  if (r <= 0) return;
  if (K % 8 || lda % 8) throw Error(ZO_ERR_DIMENSION, "extension rows must be multiples of 8");
  k_ext<<<(M + 7) / 8, 256, 0, st>>>(a, lda, M, K, bf16, Pplus, Pminus, r, rows_per_sign, ext_terms);
}

// ------------------------------------------------------------------ scored-row gather
// dst row i = src row of (sign s, sequence b, option token j) = s*B*T + b*T + prompt_len-1+j,
// i = (s*B + b)*Lopt + j: the compact rows of the last layer's pruned tail.
__global__ void k_gather_scored(const uint8_t* __restrict__ src, size_t ld_src, uint8_t* __restrict__ dst,
                                size_t ld_dst, int row_bytes, int B, int T, int prompt_len, int Lopt) {
  pdl_launch_dependents();
  pdl_wait();
  const int i = blockIdx.x;
  const int sb = i / Lopt, j = i % Lopt, sgn = sb / B, b = sb % B;
  const size_t m = (size_t)sgn * B * T + (size_t)b * T + (prompt_len - 1 + j);
  const uint4* s4 = reinterpret_cast<const uint4*>(src + m * ld_src);
  uint4* d4 = reinterpret_cast<uint4*>(dst + (size_t)i * ld_dst);
  for (int k = threadIdx.x; k < row_bytes / 16; k += blockDim.x) d4[k] = s4[k];
}

void launch_gather_scored(const void* src, size_t ld_src_bytes, void* dst, size_t ld_dst_bytes, int row_bytes,
                          int nsign, int B, int T, int prompt_len, int Lopt, cudaStream_t st) {
  if (row_bytes % 16 || ld_src_bytes % 16 || ld_dst_bytes % 16)
    throw Error(ZO_ERR_DIMENSION, "scored-row gather needs 16-byte rows");
  launch_pdl(k_gather_scored, dim3(nsign * B * Lopt), dim3(256), 0, st, static_cast<const uint8_t*>(src),
             ld_src_bytes, static_cast<uint8_t*>(dst), ld_dst_bytes, row_bytes, B, T, prompt_len, Lopt);
}

// ------------------------------------------------------------------ final LN at scored rows
// One CTA (1024 threads) per scored row: float4 loads of the row into shared memory, the
// two block reductions, xs32/xs16, then z = xs . V_e -- for r <= 8 every thread keeps r
// partial dots over its columns; above that thread (k, group) sums column k over the rows
// i = group mod G, G = 1024 / r (coalesced V_e reads), and the G group sums are added in
// group order.
constexpr int FLN_THREADS = 1024;
__global__ void __launch_bounds__(FLN_THREADS) k_final_ln(const float* __restrict__ x32, const float* __restrict__ g,
                                                         const float* __restrict__ bta, int B, int T, int d,
                                                         int prompt_len, int Lopt, float* __restrict__ xs32,
                                                         void* __restrict__ xs16, bool bf16,
                                                         const float* __restrict__ Ve, int r, float* __restrict__ z,
                                                         int rows_per_sign, long vstride) {
  extern __shared__ float sh[];
  float* row = sh;
  float* red = sh + d;  // 32 * 8 floats, then (high rank) FLN_THREADS partial dots
  const int srow = blockIdx.x;
  const int s = srow / (B * Lopt), rem = srow % (B * Lopt), b = rem / Lopt, j = rem % Lopt;
  const int m = s * B * T + b * T + (prompt_len - 1 + j);
  if (m >= rows_per_sign) {  // full scope: VectorProbe -1 copy of ln_f
    g += vstride;
    bta += vstride;
  }
  const int n4 = d >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x32 + (size_t)m * d);
  float4* row4 = reinterpret_cast<float4*>(row);
  float acc[1] = {0.f};
#pragma unroll 4
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    const float4 v = x4[i];
    row4[i] = v;
    acc[0] += (v.x + v.y) + (v.z + v.w);
  }
  block_sum<1>(acc, red);
  const float mu = acc[0] / (float)d;
  acc[0] = 0.f;
#pragma unroll 4
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    const float4 v = row4[i];
    const float a = v.x - mu, c = v.y - mu, e = v.z - mu, f = v.w - mu;
    acc[0] += (a * a + c * c) + (e * e + f * f);
  }
  block_sum<1>(acc, red);
  const float sd = sqrtf(acc[0] / (float)d + 1e-5f);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(bta);
  float4* o32 = reinterpret_cast<float4*>(xs32 + (size_t)srow * d);
#pragma unroll 4
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    const float4 v = row4[i], gg = g4[i], bb = b4[i];
    float4 h;
    h.x = (v.x - mu) / sd * gg.x + bb.x;
    h.y = (v.y - mu) / sd * gg.y + bb.y;
    h.z = (v.z - mu) / sd * gg.z + bb.z;
    h.w = (v.w - mu) / sd * gg.w + bb.w;
    row4[i] = h;
    o32[i] = h;
    store4_16(xs16, (size_t)srow * d + 4 * i, h.x, h.y, h.z, h.w, bf16);
  }
  __syncthreads();
  if (r > 8) {
    float* part = red + 32 * 8;
    const int G = blockDim.x / r, k = threadIdx.x % r, grp = threadIdx.x / r;
    float a = 0.f;
    if (threadIdx.x < G * r) {
#pragma unroll 8
      for (int i = grp; i < d; i += G) a += row[i] * Ve[(size_t)i * r + k];
    }
    part[threadIdx.x] = a;
    __syncthreads();
    if (threadIdx.x < r) {
      float t = part[threadIdx.x];
      for (int q = 1; q < G; ++q) t += part[q * r + threadIdx.x];
      z[(size_t)srow * r + threadIdx.x] = t;
    }
    return;
  }
  float a8[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a8[q] = 0.f;
#pragma unroll 4
  for (int i = threadIdx.x; i < d; i += blockDim.x)
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < r) a8[q] += row[i] * Ve[(size_t)i * r + q];
  block_sum<8>(a8, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < r; ++q) z[(size_t)srow * r + q] = a8[q];
}

void launch_final_ln(const float* x32, const float* gamma, const float* beta, int B, int T, int d, int prompt_len,
                     int Lopt, float* xs32, void* xs16, bool bf16, const float* Ve32, int r, float* z,
                     int rows_per_sign, long vstride, cudaStream_t st) {
  if (d % 4) throw Error(ZO_ERR_DIMENSION, "final LN needs dim % 4 == 0");
  if (r > FLN_THREADS) throw Error(ZO_ERR_DIMENSION, "final LN: rank above 1024");
  const size_t smem = (size_t)(d + 32 * 8 + FLN_THREADS) * sizeof(float);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    ZO_CUDA_TRY(cudaFuncSetAttribute(k_final_ln, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  k_final_ln<<<B * Lopt, FLN_THREADS, smem, st>>>(x32, gamma, beta, B, T, d, prompt_len, Lopt, xs32, xs16, bf16,
                                                    Ve32, r, z, rows_per_sign, vstride);
}

// ------------------------------------------------------------------ loss (K6b): log-softmax + gold gather
// Split-vocabulary, single pass (model.py:202-215).  Grid = (LOSS_SPLITS, scored rows):
// CTA (j, row) loads its <= LOSS_CHUNK logits of the row once into registers (float4,
// coalesced), adds the embedding LoRA term z . P_s,e[v]^T (P read once), and reduces
// them to a partial (max, sum exp(x - max)); the gold logit is captured by the CTA whose
// slice holds it.  The last CTA of a row (arrival counter) combines the partials in split
// order -- deterministic whichever CTA arrives last -- and the last row of an example sums
// its Lopt option-token NLLs in token order into nll[sign*B + b].  Counters reset
// themselves, so the launch replays inside a CUDA graph.  Probabilities are never stored.
constexpr int LOSS_THREADS = 256, LOSS_VEC = 4;  // float4 per thread per slice
constexpr int LOSS_CHUNK = LOSS_THREADS * LOSS_VEC * 4;

template <int R>
__device__ __forceinline__ float embed_term(const float* __restrict__ P, int v, const float* zs, int r) {
  float add = 0.f;
  if constexpr (R == 2) {
    const float2 p = *reinterpret_cast<const float2*>(P + (size_t)v * 2);
    add = zs[0] * p.x + zs[1] * p.y;
  } else {
    for (int k = 0; k < r; ++k) add += zs[k] * P[(size_t)v * r + k];
  }
  return add;
}

template <int R>
__global__ void __launch_bounds__(LOSS_THREADS) k_loss(const float* __restrict__ logits, int ldl, int V,
                                                       const float* __restrict__ z, int r,
                                                       const float* __restrict__ Pp, const float* __restrict__ Pm,
                                                       const int32_t* __restrict__ gold, int B, int Lopt,
                                                       float* __restrict__ part, unsigned* __restrict__ counters,
                                                       double* __restrict__ nll) {
  __shared__ float red[32];
  __shared__ float zs[8];
  __shared__ unsigned last;
  const int nsplit = gridDim.x, split = blockIdx.x, srow = blockIdx.y;
  const int ex = srow / Lopt;  // s*B + b
  const float* P = ex / B == 0 ? Pp : Pm;
  const float* lr = logits + (size_t)srow * ldl;
  const int chunk = (int)(((int64_t)V + nsplit - 1) / nsplit + 3) & ~3;
  const int v0 = split * chunk, v1 = min(V, v0 + chunk);
  const int gv = gold[srow];
  if (threadIdx.x < r) zs[threadIdx.x] = z[(size_t)srow * r + threadIdx.x];
  __syncthreads();
  float x[LOSS_VEC * 4];
  float mx = -CUDART_INF_F;
#pragma unroll
  for (int q = 0; q < LOSS_VEC; ++q) {
    const int v = v0 + 4 * (q * LOSS_THREADS + threadIdx.x);
    if (v + 3 < v1) {
      const float4 l4 = *reinterpret_cast<const float4*>(lr + v);
      x[4 * q] = l4.x, x[4 * q + 1] = l4.y, x[4 * q + 2] = l4.z, x[4 * q + 3] = l4.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) x[4 * q + e] = v + e < v1 ? lr[v + e] : -CUDART_INF_F;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (R > 0 && v + e < v1) x[4 * q + e] += embed_term<R>(P, v + e, zs, r);
      mx = fmaxf(mx, x[4 * q + e]);
      if (v + e == gv) red[31] = x[4 * q + e];  // read after the block reductions' barriers
    }
  }
  mx = block_max(mx, red);
  float acc[1] = {0.f};
#pragma unroll
  for (int q = 0; q < LOSS_VEC * 4; ++q) acc[0] += expf(x[q] - mx);
  // red[31] (the gold logit) survives: block_sum<1> writes red[warp] for 8 warps only
  const bool has_gold = gv >= v0 && gv < v1;
  const float gx = has_gold ? red[31] : 0.f;
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) {
    float* pr = part + ((size_t)srow * nsplit + split) * 2;
    pr[0] = mx;
    pr[1] = acc[0];
    if (has_gold) part[((size_t)gridDim.y * nsplit) * 2 + srow] = gx;
    __threadfence();
    last = atomicAdd(&counters[srow], 1u) == (unsigned)nsplit - 1;
  }
  __syncthreads();
  if (!last) return;
  // the row's last CTA: every slice partial is visible (fence + counter); load them in
  // parallel, combine in slice order on one thread
  __shared__ float pm[64], ps[64];
  __threadfence();
  const size_t rows_off = ((size_t)gridDim.y * nsplit) * 2 + gridDim.y;
  if (threadIdx.x < nsplit) {
    const volatile float* pv = part + ((size_t)srow * nsplit + threadIdx.x) * 2;
    pm[threadIdx.x] = pv[0];
    ps[threadIdx.x] = pv[1];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = -CUDART_INF_F;
    for (int j = 0; j < nsplit; ++j) m = fmaxf(m, pm[j]);
    float sum = 0.f;
    for (int j = 0; j < nsplit; ++j) sum += ps[j] * expf(pm[j] - m);
    const float g = ((const volatile float*)part)[((size_t)gridDim.y * nsplit) * 2 + srow];
    const float row_nll = (m + logf(sum)) - g;
    counters[srow] = 0u;
    if (Lopt == 1) {
      nll[ex] = (double)row_nll;
      return;
    }
    ((volatile float*)part)[rows_off + srow] = row_nll;
    __threadfence();
    unsigned* exc = counters + gridDim.y;
    if (atomicAdd(&exc[ex], 1u) == (unsigned)Lopt - 1) {
      __threadfence();
      float total = 0.f;
      for (int j = 0; j < Lopt; ++j) total = total + ((const volatile float*)part)[rows_off + ex * Lopt + j];
      nll[ex] = (double)total;
      exc[ex] = 0u;
    }
  }
}

// High-rank embedding delta (factorized r > 8): logits[row, v] += z[row] . P_s[v] with
// one thread per vocabulary entry holding its P row in registers for every scored row
// of its sign -- each P row is read once instead of once per scored row.
__global__ void __launch_bounds__(256) k_embed_delta(float* __restrict__ logits, int ldl, int V,
                                                     const float* __restrict__ z, int r,
                                                     const float* __restrict__ P, int row0, int nrows) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const float* pv = P + (size_t)v * r;
  for (int i = 0; i < nrows; ++i) {
    const float* zr = z + (size_t)(row0 + i) * r;
    float a = 0.f;
    for (int k = 0; k < r; k += 4) {
      const float4 p4 = *reinterpret_cast<const float4*>(pv + k);
      const float4 z4 = *reinterpret_cast<const float4*>(zr + k);
      a += p4.x * z4.x + p4.y * z4.y + p4.z * z4.z + p4.w * z4.w;
    }
    logits[(size_t)(row0 + i) * ldl + v] += a;
  }
}

size_t loss_ws_floats(int rows, int V) { return (size_t)rows * (2 * loss_splits(V) + 2); }
int loss_splits(int V) { return (int)ceil_div(V, LOSS_CHUNK); }

void launch_loss(const float* logits, int ldl, int V, const float* z, int r, const float* Pplus_e,
                 const float* Pminus_e, const int32_t* gold, int B, int Lopt, float* ws, unsigned* counters,
                 double* nll, cudaStream_t st) {
  if (ldl % 4) throw Error(ZO_ERR_DIMENSION, "logits leading dimension must be a multiple of 4");
  if (r > 8) {
    // fold the embedding's rank-r delta into the logits first, then a plain log-softmax
    if (r % 4) throw Error(ZO_ERR_DIMENSION, "high-rank embedding delta needs rank % 4 == 0");
    const int rows = B * Lopt, grid = (V + 255) / 256;
    k_embed_delta<<<grid, 256, 0, st>>>(const_cast<float*>(logits), ldl, V, z, r, Pplus_e, 0, rows);
    k_embed_delta<<<grid, 256, 0, st>>>(const_cast<float*>(logits), ldl, V, z, r, Pminus_e, rows, rows);
    r = 0;
  }
  const dim3 grid(loss_splits(V), 2 * B * Lopt);
  if (grid.x > 64) throw Error(ZO_ERR_DIMENSION, "vocabulary too large for the loss kernel's slice table");
  if (r == 0)
    k_loss<0><<<grid, LOSS_THREADS, 0, st>>>(logits, ldl, V, z, r, Pplus_e, Pminus_e, gold, B, Lopt, ws, counters, nll);
  else if (r == 2)
    k_loss<2><<<grid, LOSS_THREADS, 0, st>>>(logits, ldl, V, z, r, Pplus_e, Pminus_e, gold, B, Lopt, ws, counters, nll);
  else
    k_loss<1><<<grid, LOSS_THREADS, 0, st>>>(logits, ldl, V, z, r, Pplus_e, Pminus_e, gold, B, Lopt, ws, counters, nll);
}

// ------------------------------------------------------------------ coefficient (K7)
__device__ double pairwise_sum(const double* v, int n) {
  // numerics.py:279-284 (split at n//2, left first), iterative post-order
  if (n == 1) return v[0];
  const int h = n / 2;
  return __dadd_rn(pairwise_sum(v, h), pairwise_sum(v + h, n - h));
}

__global__ void k_coefficient(const double* __restrict__ nll, int B, double eps, double lr, int divide_by_r,
                              int rank, double* __restrict__ out4, unsigned* __restrict__ abort_flag) {
  const double lp = __ddiv_rn(pairwise_sum(nll, B), (double)B);
  const double lm = __ddiv_rn(pairwise_sum(nll + B, B), (double)B);
  const double c = __ddiv_rn(__dsub_rn(lp, lm), __dmul_rn(2.0, eps));
  const double c_used = divide_by_r ? __ddiv_rn(c, (double)rank) : c;
  const bool ok = isfinite(lp) && isfinite(lm);
  out4[0] = lp;
  out4[1] = lm;
  out4[2] = c;
  out4[3] = ok ? -__dmul_rn(lr, c_used) : 0.0;
  *abort_flag = ok ? 0u : 1u;
}

void launch_coefficient(const double* nll, int B, double eps, double lr, int divide_by_r, int rank, double* out4,
                        unsigned* abort_flag, cudaStream_t st) {
  k_coefficient<<<1, 1, 0, st>>>(nll, B, eps, lr, divide_by_r, rank, out4, abort_flag);
}

// ------------------------------------------------------------------ update (K8), probe prep
__global__ void k_update(double* __restrict__ A, const double* __restrict__ U, int64_t n,
                         const double* __restrict__ out4, const unsigned* __restrict__ abort_flag) {
  // abort_flag == nullptr: a gathered coefficient (q-direction mode) -- skip when its losses are non-finite
  if (abort_flag ? *abort_flag != 0u : !(isfinite(out4[0]) && isfinite(out4[1]))) return;
  const double beta = out4[3];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    A[i] = __dadd_rn(A[i], __dmul_rn(beta, U[i]));
}

void launch_update(double* A, const double* U, int64_t n, const double* out4, const unsigned* abort_flag,
                   cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_update<<<grid > 0 ? grid : 1, 256, 0, st>>>(A, U, n, out4, abort_flag);
}

__global__ void k_prep(const double* __restrict__ A, const double* __restrict__ U, int64_t n, double es,
                       float* __restrict__ Pp, float* __restrict__ Pm) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double a = A ? A[i] : 0.0;
    const double d = __dmul_rn(es, U[i]);
    Pp[i] = (float)__dadd_rn(a, d);
    Pm[i] = (float)__dsub_rn(a, d);
  }
}

void launch_prep_probe(const double* A, const double* U, int64_t n, double eps, double probe_scale, float* Pp,
                       float* Pm, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_prep<<<grid > 0 ? grid : 1, 256, 0, st>>>(A, U, n, eps * probe_scale, Pp, Pm);
}

// ------------------------------------------------------------------ window V -> B-operand extension columns
__global__ void k_vext(const double* __restrict__ V, int n, int r, void* __restrict__ W, int ldw, int K, bool bf16,
                       int ext_terms, float* __restrict__ V32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * r) return;
  const int j = (int)(i / r), k = (int)(i % r);
  const double v = V[i];
  const float vf = (float)v;
  if (V32) V32[i] = vf;
  if (!W) return;
  uint16_t* o = reinterpret_cast<uint16_t*>(W) + (size_t)j * ldw + K;
  if (ext_terms == 3) {
    const uint16_t hi = to16(vf, bf16);
    o[3 * k] = hi;
    o[3 * k + 1] = hi;
    o[3 * k + 2] = to16(vf - from16(hi, bf16), bf16);
  } else {
    o[k] = to16(vf, bf16);
  }
}

void launch_write_vext(const double* V, int n, int r, void* W16T, int ldw, int K, bool bf16, int ext_terms,
                       float* V32, cudaStream_t st) {
  const int64_t cnt = (int64_t)n * r;
  k_vext<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(V, n, r, W16T, ldw, K, bf16, ext_terms, V32);
}

// launch_write_vext for every matrix in one launch: the V arena is contiguous in matrix order,
// so element i belongs to the last matrix whose v_off <= i (binary search over tab)
__global__ void k_vext_all(const double* __restrict__ V, int64_t sv, const VextMat* __restrict__ tab, int ntab,
                           int r, bool bf16, int ext_terms, float* __restrict__ V32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sv) return;
  int lo = 0, hi = ntab - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (tab[mid].v_off <= i) lo = mid;
    else hi = mid - 1;
  }
  const VextMat m = tab[lo];
  const int64_t loc = i - m.v_off;
  const int j = (int)(loc / r), k = (int)(loc % r);
  const float vf = (float)V[i];
  V32[i] = vf;
  if (!m.W) return;
  uint16_t* o = reinterpret_cast<uint16_t*>(m.W) + (size_t)j * m.ldw + m.K;
  if (ext_terms == 3) {
    const uint16_t hi16 = to16(vf, bf16);
    o[3 * k] = hi16;
    o[3 * k + 1] = hi16;
    o[3 * k + 2] = to16(vf - from16(hi16, bf16), bf16);
  } else {
    o[k] = to16(vf, bf16);
  }
}

void launch_write_vext_all(const double* V, int64_t sv, const VextMat* tab, int ntab, int r, bool bf16,
                           int ext_terms, float* V32, cudaStream_t st) {
  if (sv == 0) return;
  k_vext_all<<<(unsigned)((sv + 255) / 256), 256, 0, st>>>(V, sv, tab, ntab, r, bf16, ext_terms, V32);
}

// ------------------------------------------------------------------ full-scope 1-D params (VectorProbe)
// zo_engine.py:269-295: sign +1 from 0 adds (1*eps)*z, sign -1 from +1 adds (-2*eps)*z
// (axpy_dense: product rounded, then sum), float64; the fp32 copies are what the LN
// kernels read -- [0] for the +eps rows, [1] for the -eps rows.  eps = 0 (no probe)
// makes both copies fp32(p).
__global__ void k_vec_probe(const double* __restrict__ p, const double* __restrict__ z, int64_t n, double eps,
                            float* __restrict__ out32) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (eps == 0.0 || !z) {
      out32[i] = out32[n + i] = (float)p[i];
      continue;
    }
    const double plus = __dadd_rn(p[i], __dmul_rn(eps, z[i]));
    const double minus = __dadd_rn(plus, __dmul_rn(-2.0 * eps, z[i]));
    out32[i] = (float)plus;
    out32[n + i] = (float)minus;
  }
}

void launch_vec_probe(const double* p, const double* z, int64_t n, double eps, float* out32, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  k_vec_probe<<<grid > 0 ? grid : 1, 256, 0, st>>>(p, z, n, eps, out32);
}

// VectorProbe.update (zo_engine.py:290-295): p += (-(lr*c)) * z with the UNnormalised c
// (out4[2]), skipped when the step aborted; refreshes both fp32 copies to fp32(p).
__global__ void k_vec_update(double* __restrict__ p, const double* __restrict__ z, int64_t n,
                             const double* __restrict__ out4, double lr, const unsigned* __restrict__ abort_flag,
                             float* __restrict__ out32) {
  const bool skip = abort_flag ? *abort_flag != 0u : !(isfinite(out4[0]) && isfinite(out4[1]));
  const double alpha = -__dmul_rn(lr, out4[2]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = p[i];
    if (!skip) {
      v = __dadd_rn(v, __dmul_rn(alpha, z[i]));
      p[i] = v;
    }
    out32[i] = out32[n + i] = (float)v;
  }
}

void launch_vec_update(double* p, const double* z, int64_t n, const double* out4, double lr,
                       const unsigned* abort_flag, float* out32, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  k_vec_update<<<grid > 0 ? grid : 1, 256, 0, st>>>(p, z, n, out4, lr, abort_flag, out32);
}

// ------------------------------------------------------------------ high-rank extension operand
// P16T[k][i] = h16(P[i][k]) for one matrix's [m, r] probe block: the B operand
// ([N = r, K = m], K-major) of the tensor-core extension GEMM t = a . P (r > 8).
__global__ void k_p16t(const float* __restrict__ P, int m, int r, uint16_t* __restrict__ out, bool bf16) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int yy = ty; yy < 32; yy += 8) {
    const int i = i0 + yy, k = k0 + tx;
    tile[yy][tx] = (i < m && k < r) ? P[(size_t)i * r + k] : 0.f;
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int k = k0 + yy, i = i0 + tx;
    if (i < m && k < r) out[(size_t)k * m + i] = to16(tile[tx][yy], bf16);
  }
}

void launch_p16t(const float* P, int m, int r, void* out, bool bf16, cudaStream_t st) {
  dim3 grid((m + 31) / 32, (r + 31) / 32);
  k_p16t<<<grid, dim3(32, 8), 0, st>>>(P, m, r, static_cast<uint16_t*>(out), bf16);
}

// Every extension matrix's P_s -> 16-bit [r][m] in one launch: blockIdx.x enumerates the
// 32-row tiles of all matrices (tab: per matrix {first tile, u_off, m}, ascending), y the
// 32-rank slices, z the probe sign (P+ / P- -> out / out + su).
__global__ void k_p16t_all(const float* __restrict__ Pp, const float* __restrict__ Pm, int64_t su,
                           const int64_t* __restrict__ tab, int ntab, int r, uint16_t* __restrict__ out,
                           bool bf16) {
  __shared__ float tile[32][33];
  __shared__ int64_t mat[3];
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    int lo = 0, hi = ntab - 1;  // last entry with first tile <= blockIdx.x
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (tab[3 * mid] <= (int64_t)blockIdx.x) lo = mid;
      else hi = mid - 1;
    }
    mat[0] = tab[3 * lo];
    mat[1] = tab[3 * lo + 1];
    mat[2] = tab[3 * lo + 2];
  }
  __syncthreads();
  const int m = (int)mat[2];
  const float* P = (blockIdx.z == 0 ? Pp : Pm) + mat[1];
  uint16_t* o = out + (size_t)blockIdx.z * su + mat[1];
  const int i0 = (int)((int64_t)blockIdx.x - mat[0]) * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int yy = ty; yy < 32; yy += 8) {
    const int i = i0 + yy, k = k0 + tx;
    tile[yy][tx] = (i < m && k < r) ? P[(size_t)i * r + k] : 0.f;
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int k = k0 + yy, i = i0 + tx;
    if (i < m && k < r) o[(size_t)k * m + i] = to16(tile[tx][yy], bf16);
  }
}

void launch_p16t_all(const float* Pp, const float* Pm, int64_t su, const int64_t* tab, int ntab, int tiles, int r,
                     int nsign, void* out, bool bf16, cudaStream_t st) {
  if (ntab == 0) return;
  dim3 grid((unsigned)tiles, (unsigned)((r + 31) / 32), (unsigned)nsign);
  k_p16t_all<<<grid, dim3(32, 8), 0, st>>>(Pp, Pm, su, tab, ntab, r, static_cast<uint16_t*>(out), bf16);
}

// ------------------------------------------------------------------ fold (K9) + 16-bit shadow refresh
// Low-rank (r <= 8) rewrite of a float64 master W[m, n] (reference (in, out) layout)
// and its 16-bit tensor-core copy -- HBM-bound: 8 B read (+ 8 B written) per weight
// plus the 2 B copy.  One 64 x 64 tile per CTA; warp w owns rows w, w+8, .., lane l
// columns (2l, 2l+1), so every master access is a 512 B row segment per warp
// (double2), and the transposed copy goes through a shared 16-bit tile and leaves as
// 128 B row segments.  Per-element arithmetic is numpy's (no FMA contraction):
//   LR_OUTER  axpy_outer in place (numerics.py:207-235): per k ascending
//             w = fl(w + fl(alpha * fl(l_ik * r_jk)))           (fold, dense update)
//   LR_PROBE  cached _Probe.apply (baseline_loop.py:94-98): p = dense_product (0 +
//             fl(l*r), k ascending), copy <- fl(fl(w + fl(a1*p)) [+ fl(a2*p)]); the
//             master keeps w (its bits are what restore_matrix copies back)
//   LR_DENSE  cached update: w = fl(w + fl(alpha * p))
//   LR_COPY   copy <- w (shadow refresh)
// alpha: a1 (host), fl(beta*scale) with beta = out4[3] (materialising loop), or
// fl(-fl(lr*c)*scale) with c = out4[2] (factorized update; no-op when aborted).
enum { LR_OUTER = 0, LR_PROBE = 1, LR_DENSE = 2, LR_COPY = 3 };
enum { ALPHA_HOST = 0, ALPHA_BETA = 1, ALPHA_LRC = 2 };
struct LowRankArgs {
  double* W;
  int m, n;
  const double* L;
  const double* R;
  int r;
  double a1, a2;
  const double* out4;
  double lr, scale;
  const unsigned* abort_flag;
  void* W16;
  int ldw, transposed;
  bool bf16;
  int alpha_src;
  const double* Z;  // dense direction z[m, n] (dense_mezo): p = z instead of the rank-r product
};

template <int MODE, int RK, bool DZ = false>
__global__ void __launch_bounds__(256, 3) k_lowrank(LowRankArgs a) {
  __shared__ double sL[64 * 9];
  __shared__ uint16_t t16[64 * 66];  // [j][i] 16-bit transposed tile
  double alpha = a.a1;
  if (a.alpha_src == ALPHA_BETA) {
    alpha = __dmul_rn(a.out4[3], a.scale);
  } else if (a.alpha_src == ALPHA_LRC) {
    if (a.abort_flag ? *a.abort_flag != 0u : !(isfinite(a.out4[0]) && isfinite(a.out4[1]))) return;
    alpha = __dmul_rn(-__dmul_rn(a.lr, a.out4[2]), a.scale);
  }
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = MODE == LR_COPY ? 0 : a.r;
  const int jl = 2 * lane, j = j0 + jl;
  for (int e = threadIdx.x; e < 64 * r; e += 256) {
    const int rr = e / r, k = e - rr * r;
    sL[rr * 9 + k] = (i0 + rr < a.m) ? a.L[(size_t)(i0 + rr) * r + k] : 0.0;
  }
  double rv[2][RK];  // this lane's two V rows (RK >= r; the ranks past r are never read)
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int k = 0; k < RK; ++k) rv[c][k] = (k < r && j + c < a.n) ? a.R[(size_t)(j + c) * r + k] : 0.0;
  const bool vec = (a.n & 1) == 0;
  double w[8][2], zd[8][2];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int i = i0 + warp + 8 * s;
    w[s][0] = w[s][1] = 0.0;
    zd[s][0] = zd[s][1] = 0.0;
    if (i < a.m && j < a.n) {
      const double* src = a.W + (size_t)i * a.n + j;
      if (vec) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(src));
        w[s][0] = v.x;
        w[s][1] = v.y;
      } else {
        w[s][0] = src[0];
        if (j + 1 < a.n) w[s][1] = src[1];
      }
      if (DZ) {
        const double* zs = a.Z + (size_t)i * a.n + j;
        if (vec) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(zs));
          zd[s][0] = v.x;
          zd[s][1] = v.y;
        } else {
          zd[s][0] = zs[0];
          if (j + 1 < a.n) zd[s][1] = zs[1];
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int il = warp + 8 * s;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double v = w[s][c];
      if (DZ && MODE != LR_COPY) {
        // dense direction (_DenseProbe, baseline_loop.py:107-119): axpy_dense with z itself
        if (MODE == LR_PROBE) {
          v = __dadd_rn(v, __dmul_rn(a.a1, zd[s][c]));
          if (a.a2 != 0.0) v = __dadd_rn(v, __dmul_rn(a.a2, zd[s][c]));
        } else {
          v = __dadd_rn(v, __dmul_rn(alpha, zd[s][c]));
        }
      } else if (MODE == LR_OUTER) {
#pragma unroll
        for (int k = 0; k < RK; ++k)
          if (k < r) v = __dadd_rn(v, __dmul_rn(alpha, __dmul_rn(sL[il * 9 + k], rv[c][k])));
      } else if (MODE != LR_COPY) {
        double p = 0.0;
#pragma unroll
        for (int k = 0; k < RK; ++k)
          if (k < r) p = __dadd_rn(p, __dmul_rn(sL[il * 9 + k], rv[c][k]));
        if (MODE == LR_PROBE) {
          v = __dadd_rn(v, __dmul_rn(a.a1, p));
          if (a.a2 != 0.0) v = __dadd_rn(v, __dmul_rn(a.a2, p));
        } else {
          v = __dadd_rn(v, __dmul_rn(alpha, p));
        }
      }
      w[s][c] = v;
    }
  }
  uint16_t* W16 = static_cast<uint16_t*>(a.W16);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int il = warp + 8 * s, i = i0 + il;
    if (i >= a.m || j >= a.n) continue;
    const bool two = j + 1 < a.n;
    if (MODE == LR_OUTER || MODE == LR_DENSE) {
      double* dst = a.W + (size_t)i * a.n + j;
      if (vec)
        __stcs(reinterpret_cast<double2*>(dst), make_double2(w[s][0], w[s][1]));
      else {
        dst[0] = w[s][0];
        if (two) dst[1] = w[s][1];
      }
    }
    if (!W16) continue;
    const uint16_t h0 = to16((float)w[s][0], a.bf16), h1 = to16((float)w[s][1], a.bf16);
    if (a.transposed) {
      t16[jl * 66 + il] = h0;
      t16[(jl + 1) * 66 + il] = h1;
    } else if (vec) {
      *reinterpret_cast<uint32_t*>(W16 + (size_t)i * a.n + j) = (uint32_t)h0 | ((uint32_t)h1 << 16);
    } else {
      W16[(size_t)i * a.n + j] = h0;
      if (two) W16[(size_t)i * a.n + j + 1] = h1;
    }
  }
  if (!a.transposed || !W16) return;
  __syncthreads();
  const bool v32 = (a.ldw & 1) == 0;
  const int ii = 2 * lane, io = i0 + ii;
  for (int jj = warp; jj < 64; jj += 8) {
    const int jo = j0 + jj;
    if (jo >= a.n || io >= a.m) continue;
    uint16_t* dst = W16 + (size_t)jo * a.ldw + io;
    const uint16_t x0 = t16[jj * 66 + ii], x1 = t16[jj * 66 + ii + 1];
    if (v32 && io + 1 < a.m)
      *reinterpret_cast<uint32_t*>(dst) = (uint32_t)x0 | ((uint32_t)x1 << 16);
    else {
      dst[0] = x0;
      if (io + 1 < a.m) dst[1] = x1;
    }
  }
}

template <int RK>
void launch_lowrank_rk(int mode, const LowRankArgs& a, const dim3& grid, cudaStream_t st) {
  switch (mode) {
    case LR_OUTER: k_lowrank<LR_OUTER, RK><<<grid, 256, 0, st>>>(a); break;
    case LR_PROBE: k_lowrank<LR_PROBE, RK><<<grid, 256, 0, st>>>(a); break;
    default: k_lowrank<LR_DENSE, RK><<<grid, 256, 0, st>>>(a);
  }
}

void launch_lowrank(int mode, const LowRankArgs& a, cudaStream_t st) {
  const dim3 grid((a.n + 63) / 64, (a.m + 63) / 64);
  if (a.Z && mode != LR_COPY) {
    switch (mode) {
      case LR_OUTER: k_lowrank<LR_OUTER, 1, true><<<grid, 256, 0, st>>>(a); break;
      case LR_PROBE: k_lowrank<LR_PROBE, 1, true><<<grid, 256, 0, st>>>(a); break;
      default: k_lowrank<LR_DENSE, 1, true><<<grid, 256, 0, st>>>(a);
    }
    return;
  }
  if (mode == LR_COPY || a.r == 0) {
    k_lowrank<LR_COPY, 1><<<grid, 256, 0, st>>>(a);
    return;
  }
  if (a.r <= 1) launch_lowrank_rk<1>(mode, a, grid, st);
  else if (a.r <= 2) launch_lowrank_rk<2>(mode, a, grid, st);
  else if (a.r <= 4) launch_lowrank_rk<4>(mode, a, grid, st);
  else launch_lowrank_rk<8>(mode, a, grid, st);
}

LowRankArgs lowrank_args(double* W64, int m, int n, const double* L, const double* R, int r, void* W16, int ldw,
                         int transposed, bool bf16) {
  LowRankArgs a{};
  a.W = W64;
  a.m = m;
  a.n = n;
  a.L = L;
  a.R = R;
  a.r = r;
  a.W16 = W16;
  a.ldw = ldw;
  a.transposed = transposed;
  a.bf16 = bf16;
  a.scale = 1.0;
  a.alpha_src = ALPHA_HOST;
  return a;
}

// High-rank variant (factorized r > 8, e.g. BASELINE config 5's r = 128 where this is
// the dominant cost of a step: 3 float64 ops per weight per rank).  64x64 W tile per CTA,
// each thread a 4x4 register micro-tile; the tile's A rows and V rows are staged
// through shared memory 32 ranks at a time (V transposed).  Same per-element
// arithmetic and order as k_lowrank LR_OUTER: w = w + alpha*(A_ik*V_jk), k ascending.
__global__ void __launch_bounds__(256) k_fold_dev_tiled(double* __restrict__ W, int m, int n,
                                                        const double* __restrict__ A, const double* __restrict__ Vv,
                                                        int r, const double* __restrict__ out4, double lr,
                                                        double scale, const unsigned* __restrict__ abort_flag,
                                                        void* __restrict__ W16, int ldw, int transposed, bool bf16,
                                                        double alpha_fixed) {
  // out4 == nullptr: a host-side alpha (zo_update_dense / window fold); else alpha from the
  // device coefficient, skipped when the step aborted
  double alpha = alpha_fixed;
  if (out4) {
    if (abort_flag ? *abort_flag != 0u : !(isfinite(out4[0]) && isfinite(out4[1]))) return;
    alpha = __dmul_rn(-__dmul_rn(lr, out4[2]), scale);
  }
  __shared__ double smem[64 * 33 + 32 * 65];
  double* sA = smem;             // [64 rows i][33]: k within the chunk
  double* sVt = smem + 64 * 33;  // [32 k][65]: column j
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16
  double w[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      w[a][b] = (i < m && j < n) ? W[(size_t)i * n + j] : 0.0;
    }
  for (int k0 = 0; k0 < r; k0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int rr = e >> 5, k = e & 31;
      sA[rr * 33 + k] = (i0 + rr < m && k0 + k < r) ? A[(size_t)(i0 + rr) * r + k0 + k] : 0.0;
      sVt[k * 65 + rr] = (j0 + rr < n && k0 + k < r) ? Vv[(size_t)(j0 + rr) * r + k0 + k] : 0.0;
    }
    __syncthreads();
    const int kn = min(32, r - k0);
    for (int k = 0; k < kn; ++k) {
      double av[4], vv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sA[(ty + 16 * a) * 33 + k];
#pragma unroll
      for (int b = 0; b < 4; ++b) vv[b] = sVt[k * 65 + tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) w[a][b] = __dadd_rn(w[a][b], __dmul_rn(alpha, __dmul_rn(av[a], vv[b])));
    }
  }
  __syncthreads();
  float* tile = reinterpret_cast<float*>(smem);  // [64][65] fp32 image for the transposed shadow
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int yy = ty + 16 * a, xx = tx + 16 * b, i = i0 + yy, j = j0 + xx;
      float f = 0.f;
      if (i < m && j < n) {
        W[(size_t)i * n + j] = w[a][b];
        f = (float)w[a][b];
        if (!transposed && W16) reinterpret_cast<uint16_t*>(W16)[(size_t)i * n + j] = to16(f, bf16);
      }
      tile[yy * 65 + xx] = f;
    }
  if (!transposed || !W16) return;
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int jj = e >> 6, ii = e & 63, j = j0 + jj, i = i0 + ii;
    if (i < m && j < n) reinterpret_cast<uint16_t*>(W16)[(size_t)j * ldw + i] = to16(tile[ii * 65 + jj], bf16);
  }
}

void launch_fold_dev(double* W64, int m, int n, const double* A, const double* V, int r, const double* out4,
                     double lr, double scale, const unsigned* abort_flag, void* W16, int ldw, int transposed,
                     bool bf16, cudaStream_t st) {
  if (r > 8) {
    k_fold_dev_tiled<<<dim3((n + 63) / 64, (m + 63) / 64), 256, 0, st>>>(W64, m, n, A, V, r, out4, lr, scale,
                                                                          abort_flag, W16, ldw, transposed, bf16, 0.0);
    return;
  }
  LowRankArgs a = lowrank_args(W64, m, n, A, V, r, W16, ldw, transposed, bf16);
  a.out4 = out4;
  a.lr = lr;
  a.scale = scale;
  a.abort_flag = abort_flag;
  a.alpha_src = ALPHA_LRC;
  launch_lowrank(LR_OUTER, a, st);
}

void launch_fold(double* W64, int m, int n, const double* A, const double* V, int r, double alpha, void* W16,
                 int ldw, int transposed, bool bf16, cudaStream_t st) {
  if (r > 8) {
    k_fold_dev_tiled<<<dim3((n + 63) / 64, (m + 63) / 64), 256, 0, st>>>(W64, m, n, A, V, r, nullptr, 0.0, 0.0,
                                                                          nullptr, W16, ldw, transposed, bf16, alpha);
    return;
  }
  LowRankArgs a = lowrank_args(W64, m, n, A, V, r, W16, ldw, transposed, bf16);
  a.a1 = alpha;
  launch_lowrank(LR_OUTER, a, st);
}

void launch_shadow_T(const double* W64, int m, int n, void* W16T, int ldw, bool bf16, cudaStream_t st) {
  launch_lowrank(LR_COPY, lowrank_args(const_cast<double*>(W64), m, n, nullptr, nullptr, 0, W16T, ldw, 1, bf16), st);
}

__global__ void k_shadow(const double* __restrict__ W, int64_t count, void* __restrict__ o, bool bf16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    reinterpret_cast<uint16_t*>(o)[i] = to16((float)W[i], bf16);
}

void launch_shadow(const double* W64, int64_t count, void* W16, bool bf16, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 16);
  k_shadow<<<grid > 0 ? grid : 1, 256, 0, st>>>(W64, count, W16, bf16);
}

__global__ void k_f64_to_f32(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = (float)a[i];
}
void launch_f64_to_f32(const double* a, float* b, int64_t n, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_f64_to_f32<<<grid > 0 ? grid : 1, 256, 0, st>>>(a, b, n);
}

__global__ void k_f32_to_f64(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = (double)a[i];
}
void launch_f32_to_f64(const float* a, double* b, int64_t n, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_f32_to_f64<<<grid > 0 ? grid : 1, 256, 0, st>>>(a, b, n);
}

void launch_zero(void* p, size_t bytes, cudaStream_t st) { ZO_CUDA_TRY(cudaMemsetAsync(p, 0, bytes, st)); }

// ------------------------------------------------------------------ materialising-loop comparand
// baseline_loop.py:68-119 / 122-239: the conventional training loop writes every
// perturbed matrix four times per step.  One 64x64 W tile per CTA, 4x4 per thread,
// U/V rows staged through shared memory 32 ranks at a time.
//   BL_PROBE   (cached _Probe.apply): P = dense_product(U, V) (numerics.py:256-267:
//              0 + fl(u*v), k ascending), w = fl(w0 + fl(a1*P)) [then fl(w + fl(a2*P))]
//              -> the 16-bit serving copy only.  The float64 master keeps w0, which is
//              exactly the bits restore_matrix copies back (numerics.py:246-253).
//   BL_UPDATE  (cached update): alpha = fl(beta*scale) from the device coefficient,
//              w = fl(w0 + fl(alpha*P)) -> master + 16-bit copy.
//   BL_OUTER   (recompute mode, axpy_outer in place, numerics.py:207-235): per k
//              w = fl(w + fl(alpha*fl(u*v))) -> master + 16-bit copy; alpha = a1, or
//              fl(beta*scale) when out4 is given.
enum { BL_PROBE = 0, BL_UPDATE = 1, BL_OUTER = 2 };

template <int MODE>
__global__ void __launch_bounds__(256) k_materialise(double* __restrict__ W, int m, int n,
                                                     const double* __restrict__ U, const double* __restrict__ Vv,
                                                     int r, double a1, double a2, const double* __restrict__ out4,
                                                     double scale, void* __restrict__ W16, int ldw, int transposed,
                                                     bool bf16) {
  double alpha = a1;
  if (out4) alpha = __dmul_rn(out4[3], scale);
  __shared__ double smem[64 * 33 + 32 * 65];
  double* sU = smem;             // [64 rows i][33]
  double* sVt = smem + 64 * 33;  // [32 k][65]
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double w[4][4], p[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      w[a][b] = (i < m && j < n) ? W[(size_t)i * n + j] : 0.0;
      p[a][b] = 0.0;
    }
  for (int k0 = 0; k0 < r; k0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int rr = e >> 5, k = e & 31;
      sU[rr * 33 + k] = (i0 + rr < m && k0 + k < r) ? U[(size_t)(i0 + rr) * r + k0 + k] : 0.0;
      sVt[k * 65 + rr] = (j0 + rr < n && k0 + k < r) ? Vv[(size_t)(j0 + rr) * r + k0 + k] : 0.0;
    }
    __syncthreads();
    const int kn = min(32, r - k0);
    for (int k = 0; k < kn; ++k) {
      double uv[4], vv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) uv[a] = sU[(ty + 16 * a) * 33 + k];
#pragma unroll
      for (int b = 0; b < 4; ++b) vv[b] = sVt[k * 65 + tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double t = __dmul_rn(uv[a], vv[b]);
          if (MODE == BL_OUTER)
            w[a][b] = __dadd_rn(w[a][b], __dmul_rn(alpha, t));
          else
            p[a][b] = __dadd_rn(p[a][b], t);
        }
    }
  }
  __syncthreads();
  float* tile = reinterpret_cast<float*>(smem);  // [64][65] fp32 image for the transposed copy
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int yy = ty + 16 * a, xx = tx + 16 * b, i = i0 + yy, j = j0 + xx;
      double v = w[a][b];
      if (MODE == BL_PROBE) {
        v = __dadd_rn(v, __dmul_rn(a1, p[a][b]));
        if (a2 != 0.0) v = __dadd_rn(v, __dmul_rn(a2, p[a][b]));
      } else if (MODE == BL_UPDATE) {
        v = __dadd_rn(v, __dmul_rn(alpha, p[a][b]));
      }
      float f = 0.f;
      if (i < m && j < n) {
        if (MODE != BL_PROBE) W[(size_t)i * n + j] = v;
        f = (float)v;
        if (!transposed && W16) reinterpret_cast<uint16_t*>(W16)[(size_t)i * n + j] = to16(f, bf16);
      }
      tile[yy * 65 + xx] = f;
    }
  if (!transposed || !W16) return;
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int jj = e >> 6, ii = e & 63, j = j0 + jj, i = i0 + ii;
    if (i < m && j < n) reinterpret_cast<uint16_t*>(W16)[(size_t)j * ldw + i] = to16(tile[ii * 65 + jj], bf16);
  }
}

void launch_materialise(int mode, double* W64, int m, int n, const double* U, const double* V, int r, double a1,
                        double a2, const double* out4, double scale, void* W16, int ldw, int transposed, bool bf16,
                        cudaStream_t st) {
  if (r <= 8) {  // HBM-bound: the row-segment kernel
    LowRankArgs a = lowrank_args(W64, m, n, U, V, r, W16, ldw, transposed, bf16);
    a.a1 = a1;
    a.a2 = a2;
    a.out4 = out4;
    a.scale = scale;
    a.alpha_src = out4 ? ALPHA_BETA : ALPHA_HOST;
    launch_lowrank(mode == BL_PROBE ? LR_PROBE : mode == BL_UPDATE ? LR_DENSE : LR_OUTER, a, st);
    return;
  }
  const dim3 grid((n + 63) / 64, (m + 63) / 64);
  switch (mode) {
    case BL_PROBE:
      k_materialise<BL_PROBE><<<grid, 256, 0, st>>>(W64, m, n, U, V, r, a1, a2, nullptr, scale, W16, ldw,
                                                    transposed, bf16);
      break;
    case BL_UPDATE:
      k_materialise<BL_UPDATE><<<grid, 256, 0, st>>>(W64, m, n, U, V, r, 0.0, 0.0, out4, scale, W16, ldw,
                                                     transposed, bf16);
      break;
    default:
      k_materialise<BL_OUTER><<<grid, 256, 0, st>>>(W64, m, n, U, V, r, a1, 0.0, out4, scale, W16, ldw,
                                                    transposed, bf16);
  }
}

void launch_dense_rw(int mode, double* W64, int m, int n, const double* Z, double a1, double a2, const double* out4,
                     void* W16, int ldw, int transposed, bool bf16, cudaStream_t st) {
  LowRankArgs a = lowrank_args(W64, m, n, nullptr, nullptr, 0, W16, ldw, transposed, bf16);
  a.Z = Z;
  a.a1 = a1;
  a.a2 = a2;
  a.out4 = out4;
  a.alpha_src = out4 ? ALPHA_BETA : ALPHA_HOST;
  launch_lowrank(mode == BL_PROBE ? LR_PROBE : mode == BL_UPDATE ? LR_DENSE : mode == 3 ? LR_COPY : LR_OUTER, a, st);
}

// _DenseProbe on 1-D params in recompute mode (in place): p = fl(p + fl(alpha*z)),
// alpha = a1 or beta from the device coefficient; both fp32 copies refreshed
__global__ void k_vec_inplace(double* __restrict__ p, const double* __restrict__ z, int64_t n, double a1,
                              const double* __restrict__ out4, float* __restrict__ out32) {
  const double alpha = out4 ? out4[3] : a1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = __dadd_rn(p[i], __dmul_rn(alpha, z[i]));
    p[i] = v;
    out32[i] = out32[n + i] = (float)v;
  }
}

void launch_vec_inplace(double* p, const double* z, int64_t n, double a1, const double* out4, float* out32,
                        cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  k_vec_inplace<<<grid > 0 ? grid : 1, 256, 0, st>>>(p, z, n, a1, out4, out32);
}

// VectorProbe.set_sign for ONE scoring call (the loop scores each sign separately):
// both fp32 copies = fp32(p + eps*z) (sign +1) or fp32((p + eps*z) + (-2 eps)*z) (sign -1)
__global__ void k_vec_probe_sign(const double* __restrict__ p, const double* __restrict__ z, int64_t n, double eps,
                                 int sign, float* __restrict__ out32) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = __dadd_rn(p[i], __dmul_rn(eps, z[i]));
    if (sign < 0) v = __dadd_rn(v, __dmul_rn(-2.0 * eps, z[i]));
    out32[i] = out32[n + i] = (float)v;
  }
}

void launch_vec_probe_sign(const double* p, const double* z, int64_t n, double eps, int sign, float* out32,
                           cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  k_vec_probe_sign<<<grid > 0 ? grid : 1, 256, 0, st>>>(p, z, n, eps, sign, out32);
}

}  // namespace zo
