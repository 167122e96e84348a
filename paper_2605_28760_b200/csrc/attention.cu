// K3 -- small-T causal attention per (sequence, head) (model.py:184-194).
//
// T <= 128 tokens and dh in {16, 32, 64, 128}: one CTA of ceil(T/16) warps per
// (sequence, head); Q, K, V (16-bit, from the packed qkv GEMM output) are
// staged in shared memory with 16-byte loads, S = Q K^T and O = P V run on the
// tensor cores (mma.sync m16n8k16, fp32 accumulate) with the causal softmax
// kept in registers between them (the S accumulator fragment is re-used as the
// A fragment of P V).  Warp w owns query rows [16w, 16w+16) and only visits
// key blocks <= its own (causal).  FLOPs are <0.3% of the step; the kernel is
// bound by reading qkv once (HBM) -- the SIMT version was 35% of the step.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "zo_common.cuh"
#include "zo_kernels.h"

namespace zo {

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
template <bool BF16>
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  if constexpr (BF16) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}
template <bool BF16>
__device__ __forceinline__ float unpack_f(uint32_t w, int hi) {
  const uint16_t h = (uint16_t)(w >> (16 * hi));
  if constexpr (BF16) return __bfloat162float(__ushort_as_bfloat16(h));
  else return __half2float(__ushort_as_half(h));
}
template <bool BF16>
__device__ __forceinline__ uint32_t pack_f2(float a, float b) {
  if constexpr (BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

// One warp's 16 query rows [r0, r0+16) against its KB causal key blocks (compile-time,
// so the score / probability fragments stay in registers with no runtime masks outside
// the diagonal block); XR = fused LoRA-extension rank (0: none).
template <int DH, int KB, bool BF16, int XR>
__device__ __forceinline__ void attn_rows(const uint16_t* sq, const uint16_t* sk, const uint16_t* sv, const float* sP,
                                          uint16_t* __restrict__ ctx, int ldc, int T, int seq, int h, int r0,
                                          const AttnExt& x) {
  constexpr int LD = DH + 8;
  constexpr int NT = 2 * KB;  // key n-tiles of 8
  constexpr int DT = DH / 8;  // output n-tiles
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const uint32_t sq_a = static_cast<uint32_t>(__cvta_generic_to_shared(sq));
  const uint32_t sk_a = static_cast<uint32_t>(__cvta_generic_to_shared(sk));
  const uint32_t sv_a = static_cast<uint32_t>(__cvta_generic_to_shared(sv));
  float s[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    uint32_t a0, a1, a2, a3;
    ldsm_x4(sq_a + 2 * ((r0 + (lane & 15)) * LD + kk * 16 + (lane >> 4) * 8), a0, a1, a2, a3);
#pragma unroll
    for (int nb = 0; nb < KB; ++nb) {
      uint32_t b0, b1, b2, b3;
      const int q = lane >> 3;
      ldsm_x4(sk_a + 2 * ((nb * 16 + (q >> 1) * 8 + (lane & 7)) * LD + kk * 16 + (q & 1) * 8), b0, b1, b2, b3);
      mma16816<BF16>(s[2 * nb], a0, a1, a2, a3, b0, b1);
      mma16816<BF16>(s[2 * nb + 1], a0, a1, a2, a3, b2, b3);
    }
  }
  // causal softmax on the fragments (rows r0+g, r0+g+8; cols 8n + 2tq (+1)), base-2 with
  // the 1/sqrt(dh) scale folded into the exponent; only the diagonal block is masked
  const float sl2 = rsqrtf((float)DH) * 1.4426950408889634f;
  float mx[2] = {-CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
  for (int n = 0; n < NT; ++n) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float v = s[n][e] * sl2;
      if (n >= NT - 2) {
        const int row = r0 + g + ((e >> 1) << 3), col = n * 8 + 2 * tq + (e & 1);
        if (col > row || col >= T) v = -CUDART_INF_F;
      }
      s[n][e] = v;
      mx[e >> 1] = fmaxf(mx[e >> 1], v);
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
    mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
  }
  float sum[2] = {0.f, 0.f};
#pragma unroll
  for (int n = 0; n < NT; ++n) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float p = exp2f(s[n][e] - mx[e >> 1]);  // exp2(-inf) = 0 for masked entries
      s[n][e] = p;
      sum[e >> 1] += p;
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    sum[i] += __shfl_xor_sync(0xffffffffu, sum[i], 1);
    sum[i] += __shfl_xor_sync(0xffffffffu, sum[i], 2);
  }
  // O = P V
  float o[DT][4];
#pragma unroll
  for (int n = 0; n < DT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < KB; ++kp) {
    const uint32_t a0 = pack_f2<BF16>(s[2 * kp][0], s[2 * kp][1]);
    const uint32_t a1 = pack_f2<BF16>(s[2 * kp][2], s[2 * kp][3]);
    const uint32_t a2 = pack_f2<BF16>(s[2 * kp + 1][0], s[2 * kp + 1][1]);
    const uint32_t a3 = pack_f2<BF16>(s[2 * kp + 1][2], s[2 * kp + 1][3]);
#pragma unroll
    for (int nc = 0; nc < DT / 2; ++nc) {
      uint32_t b0, b1, b2, b3;
      const int q = lane >> 3;
      ldsm_x4_t(sv_a + 2 * ((kp * 16 + (q & 1) * 8 + (lane & 7)) * LD + nc * 16 + (q >> 1) * 8), b0, b1, b2, b3);
      mma16816<BF16>(o[2 * nc], a0, a1, a2, a3, b0, b1);
      mma16816<BF16>(o[2 * nc + 1], a0, a1, a2, a3, b2, b3);
    }
  }
  const float inv0 = 1.f / sum[0], inv1 = 1.f / sum[1];
  const int row0 = r0 + g, row1 = r0 + g + 8;
  const int m0 = seq * T + row0, m1 = seq * T + row1;
  // XR = 8 also serves ranks 3, 5, 6, 7 (runtime rank x.r, compile-time bound 8)
  constexpr int XK = XR > 0 ? XR : 1;
  const int xs = XR == 8 ? x.r : XR;  // rank = row stride of P
  float t0[XK], t1[XK];
#pragma unroll
  for (int k = 0; k < XK; ++k) t0[k] = t1[k] = 0.f;
#pragma unroll
  for (int n = 0; n < DT; ++n) {
    const int col = h * DH + n * 8 + 2 * tq;
    const int lc = n * 8 + 2 * tq;  // column within the head (index into sP)
    const uint32_t w0 = pack_f2<BF16>(o[n][0] * inv0, o[n][1] * inv0);
    const uint32_t w1 = pack_f2<BF16>(o[n][2] * inv1, o[n][3] * inv1);
    if (row0 < T) *reinterpret_cast<uint32_t*>(ctx + (size_t)m0 * ldc + col) = w0;
    if (row1 < T) *reinterpret_cast<uint32_t*>(ctx + (size_t)m1 * ldc + col) = w1;
    if constexpr (XR > 0) {
      // partial LoRA-extension dots of the stored ctx with the attn_out P+- (model.py:191-192)
      const float a00 = unpack_f<BF16>(w0, 0), a01 = unpack_f<BF16>(w0, 1);
      const float a10 = unpack_f<BF16>(w1, 0), a11 = unpack_f<BF16>(w1, 1);
#pragma unroll
      for (int k = 0; k < XR; ++k) {
        if (XR == 8 && k >= xs) break;
        const float pa = sP[lc * xs + k], pb = sP[(lc + 1) * xs + k];
        t0[k] += a00 * pa + a01 * pb;
        t1[k] += a10 * pa + a11 * pb;
      }
    }
  }
  if constexpr (XR > 0) {
#pragma unroll
    for (int k = 0; k < XR; ++k) {
      t0[k] += __shfl_xor_sync(0xffffffffu, t0[k], 1);
      t0[k] += __shfl_xor_sync(0xffffffffu, t0[k], 2);
      t1[k] += __shfl_xor_sync(0xffffffffu, t1[k], 1);
      t1[k] += __shfl_xor_sync(0xffffffffu, t1[k], 2);
    }
    if (tq == 0) {
#pragma unroll
      for (int k = 0; k < XR; ++k) {
        if (XR == 8 && k >= xs) break;
        if (row0 < T) x.tpart[((size_t)h * x.ld + m0) * xs + k] = t0[k];
        if (row1 < T) x.tpart[((size_t)h * x.ld + m1) * xs + k] = t1[k];
      }
    }
  }
}

template <int DH, int TP, bool BF16, int XR>
__global__ void __launch_bounds__(TP * 2)
    k_attn_mma(const uint16_t* __restrict__ qkv, int ldq, uint16_t* __restrict__ ctx, int ldc, int T, int H,
               AttnExt x) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int LD = DH + 8;  // padded row (halves): conflict-free ldmatrix
  extern __shared__ __align__(16) uint16_t sm[];
  uint16_t* sq = sm;
  uint16_t* sk = sq + TP * LD;
  uint16_t* sv = sk + TP * LD;
  float* sP = reinterpret_cast<float*>(sv + TP * LD);  // this head's P rows [DH][r] (one sign per sequence)
  const int seq = blockIdx.x, h = blockIdx.y;
  const int d = H * DH;
  if constexpr (XR > 0) {
    const int xs = XR == 8 ? x.r : XR;
    const float* Pg = ((seq * T) < x.rps ? x.Pp : x.Pm) + (size_t)h * DH * xs;
    for (int i = threadIdx.x; i < DH * xs; i += blockDim.x) sP[i] = Pg[i];
  }
  // stage Q, K, V with asynchronous 16-byte copies (cp.async): every load of the CTA is
  // in flight at once instead of one dependent load/store round trip per row block
  // (the kernel is bound by this read of qkv); rows >= T are zero-filled
  constexpr int VPR = DH / 8;
  for (int idx = threadIdx.x; idx < TP * VPR; idx += blockDim.x) {
    const int t = idx / VPR, c = (idx % VPR) * 8;
    const uint32_t dq = static_cast<uint32_t>(__cvta_generic_to_shared(sq + t * LD + c));
    const uint32_t dk = static_cast<uint32_t>(__cvta_generic_to_shared(sk + t * LD + c));
    const uint32_t dv = static_cast<uint32_t>(__cvta_generic_to_shared(sv + t * LD + c));
    const uint16_t* src = qkv + (size_t)(seq * T + (t < T ? t : 0)) * ldq + (size_t)h * DH + c;
    const int nbytes = t < T ? 16 : 0;  // src-size 0: the 16 bytes are zero-filled
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dq), "l"(src), "r"(nbytes) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dk), "l"(src + d), "r"(nbytes) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dv), "l"(src + 2 * d), "r"(nbytes)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int r0 = warp * 16;
  if (r0 >= T) return;
  // warp w owns query rows [16w, 16w+16) and the key blocks 0..w (causal)
  switch (warp) {
    case 0: attn_rows<DH, 1, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x); break;
    case 1: attn_rows<DH, 2, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x); break;
    case 2: if constexpr (TP >= 64) attn_rows<DH, 3, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x); break;
    case 3: if constexpr (TP >= 64) attn_rows<DH, 4, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x); break;
    case 4: if constexpr (TP >= 128) attn_rows<DH, 5, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x); break;
    case 5: if constexpr (TP >= 128) attn_rows<DH, 6, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x); break;
    case 6: if constexpr (TP >= 128) attn_rows<DH, 7, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x); break;
    default: if constexpr (TP >= 128) attn_rows<DH, 8, BF16, XR>(sq, sk, sv, sP, ctx, ldc, T, seq, h, r0, x);
  }
}

template <int DH, int TP, bool BF16, int XR>
static void launch_t(const void* qkv, int ldq, void* ctx, int ldc, int nseq, int T, int H, const AttnExt& x,
                     cudaStream_t st) {
  const size_t smem = (size_t)3 * TP * (DH + 8) * 2 + (size_t)DH * 8 * sizeof(float);
  static bool set = false;
  if (!set) {
    ZO_CUDA_TRY(cudaFuncSetAttribute(k_attn_mma<DH, TP, BF16, XR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    set = true;
  }
  launch_pdl(k_attn_mma<DH, TP, BF16, XR>, dim3(nseq, H), dim3(TP * 2), smem, st,
             static_cast<const uint16_t*>(qkv), ldq, static_cast<uint16_t*>(ctx), ldc, T, H, x);
}

template <int DH, int TP, bool BF16>
static void launch_xr(const void* qkv, int ldq, void* ctx, int ldc, int nseq, int T, int H, const AttnExt& x,
                      cudaStream_t st) {
  switch (x.tpart ? x.r : 0) {
    case 0: launch_t<DH, TP, BF16, 0>(qkv, ldq, ctx, ldc, nseq, T, H, x, st); return;
    case 1: launch_t<DH, TP, BF16, 1>(qkv, ldq, ctx, ldc, nseq, T, H, x, st); return;
    case 2: launch_t<DH, TP, BF16, 2>(qkv, ldq, ctx, ldc, nseq, T, H, x, st); return;
    case 4: launch_t<DH, TP, BF16, 4>(qkv, ldq, ctx, ldc, nseq, T, H, x, st); return;
    default: launch_t<DH, TP, BF16, 8>(qkv, ldq, ctx, ldc, nseq, T, H, x, st); return;  // 3, 5..8
  }
}

template <int DH, bool BF16>
static void launch_dh(const void* qkv, int ldq, void* ctx, int ldc, int nseq, int T, int H, const AttnExt& x,
                      cudaStream_t st) {
  if (T <= 32) launch_xr<DH, 32, BF16>(qkv, ldq, ctx, ldc, nseq, T, H, x, st);
  else if (T <= 64) launch_xr<DH, 64, BF16>(qkv, ldq, ctx, ldc, nseq, T, H, x, st);
  else launch_xr<DH, 128, BF16>(qkv, ldq, ctx, ldc, nseq, T, H, x, st);
}

void launch_attention(const void* qkv, int ldq, void* ctx, int ldc, int nseq, int T, int H, int dh, bool bf16,
                      const AttnExt& x, cudaStream_t st) {
  if (x.tpart && (x.r < 1 || x.r > 8)) throw Error(ZO_ERR_DIMENSION, "fused attention extension needs 1 <= r <= 8");
  if (T > 128) throw Error(ZO_ERR_DIMENSION, "attention kernel supports T <= 128");
  if (ldq % 8 || ldc % 2) throw Error(ZO_ERR_DIMENSION, "attention operands must be 16-byte aligned");
#define ZO_DH(D)                                                                    \
  case D:                                                                           \
    if (bf16) launch_dh<D, true>(qkv, ldq, ctx, ldc, nseq, T, H, x, st);             \
    else launch_dh<D, false>(qkv, ldq, ctx, ldc, nseq, T, H, x, st);                 \
    return;
  switch (dh) {
    ZO_DH(16)
    ZO_DH(32)
    ZO_DH(64)
    ZO_DH(128)
    default: throw Error(ZO_ERR_DIMENSION, "head dim must be 16, 32, 64 or 128");
  }
#undef ZO_DH
}

}  // namespace zo
