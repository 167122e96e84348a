// K2 -- persistent tcgen05 GEMM for sm_100a.
//
// Roles (192 threads, 1 CTA/SM):
//   warp 0      TMA producer: A/B tiles (SWIZZLE_128B, K-major) into a STAGES-deep
//               shared-memory ring, completion via mbarrier transaction bytes.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (kind::f16, M=128, N=BN, K=16 per instruction, fp32 accumulate
//               in TMEM); tcgen05.commit frees smem stages / publishes tiles.
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> fused op -> HBM.
// Two TMEM accumulators (2*BN columns) let the epilogue of tile i overlap the
// MMAs of tile i+1.  Tiles are scheduled M-fastest so the CTAs resident at
// once share weight (B) tiles through L2: every weight byte crosses HBM once
// per launch for both perturbation signs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "zo_common.cuh"
#include "zo_gemm.h"

namespace zo {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  // bounded spin: a protocol bug traps (kernel error) instead of hanging the GPU
  for (uint32_t i = 0;; ++i) {
    uint32_t done;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (i > (1u << 26)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-CTA TMA: both CTAs' bytes complete on the leader CTA's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_commit_cg2(uint32_t bar) {
  // arrive on the barrier at this offset in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
template <bool TF32>
__device__ __forceinline__ void tc_mma_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accum) {
  if constexpr (TF32)
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
  else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// relaxed arrives: the barrier orders only what the waiting side needs (TMEM reads fenced by
// tcgen05.fence::before_thread_sync, shared-memory reads whose values are already in
// registers), not the arriving warp's outstanding global stores -- a release arrive waits
// for those to be acknowledged (ERRBAR), once per tile per warp
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(cta));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_arrive_relaxed(uint32_t bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
template <bool TF32>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  if constexpr (TF32)
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
  else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
// K-major, 128-byte swizzle, 8-row core groups 1024 B apart (sm_100 descriptor, version 1).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;            // version
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float gelu_tanh(float x) {
  // model.py:145-146: 0.5*x*(1 + tanh(sqrt(2/pi)*(x + 0.044715*x^3))), evaluated as the
  // identity 0.5*(1 + tanh(u)) = 1/(1 + e^(-2u)): one ex2 + one reciprocal on the SFU
  // instead of tanhf's polynomial/branch sequence (abs. error of 0.5*(1+tanh) ~1e-7,
  // far below the 16-bit rounding of the stored activation)
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  return __fdividef(x, 1.0f + __expf(-2.0f * u));
}

template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

template <bool BF16>
__device__ __forceinline__ float unpack16(uint32_t w, int hi) {
  const uint16_t h = (uint16_t)(w >> (16 * hi));
  if constexpr (BF16) return __bfloat162float(__ushort_as_bfloat16(h));
  else return __half2float(__ushort_as_half(h));
}

template <int BN, int CG = 1, bool UPD = false, bool OBOX = false>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;  // rows per CTA; a CTA pair (CG = 2) covers 256
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // EPI_UPDATE32: a short operand ring (K = rank) and a ring of fp32 master blocks
  // [32 rows][128 cols] TMA-loaded (8 x 16 KB in flight); even slot count: a slot always serves
  // the same epilogue warp group
  static constexpr int W_SLOTS = UPD ? 8 : 0;
  static constexpr int W_BYTES = 32 * BM * 4;
  // OBOX (the residual and 16-bit-output epilogues): 32 KB of 4 KB staging boxes for the TMA
  // stores -- per epilogue warp two 32 x 32 fp32 boxes (the residual reduce-add) or 32 x 64
  // 16-bit boxes (two per warp with one epilogue group, one with two) -- paid for with one
  // operand stage when the ring would not fit beside them
  static constexpr int O_BYTES = OBOX ? 4 * 2 * 32 * 32 * 4 : 0;
  static constexpr int STAGES_MAX = (196 * 1024) / STAGE_BYTES > 8 ? 8 : (196 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = UPD ? 3 : (OBOX && STAGES_MAX * STAGE_BYTES + O_BYTES > 200 * 1024 ? STAGES_MAX - 1 : STAGES_MAX);
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + W_SLOTS * W_BYTES + O_BYTES + 512;
};

struct GemmParams {
  int M, N, num_kb, last_ksteps, m_tiles, n_tiles, ldo;
  int kb0;  // first K block of this launch (the tf32 path's K-chunked launches; 0 otherwise)
  void* out;
  // EPI_GELU16_EXT: per-tile partial LoRA-extension dots of the stored 16-bit
  // activation with the NEXT matrix's P+- (see zo_gemm.h)
  const float* xPp;
  const float* xPm;
  int xr, xrps, tpart_ld;
  float* tpart;
  // stream-K tail (sk = 1): unit u (a CTA, or a CTA pair when CG = 2) owns the global
  // k-iterations [sk_dp*num_kb + u*sk_w, +sk_w) of the tiles past the data-parallel
  // waves.  A segment that starts after the tile's first k-block publishes its fp32
  // partial (sk_ws / sk_flags slot of its CTA); the unit holding the first k-block owns
  // the epilogue: its accumulator + the later units' partials in ascending k order --
  // a fixed summation order, independent of timing.
  int sk, sk_w, sk_dp;
  float* sk_ws;
  unsigned* sk_flags;
  int half_dp, half_n;  // half-width tail tiles (see zo_gemm.h)
  // split-K (gemm_enable_splitk): CTA u computes k-blocks [s*kchunk, +kchunk) of tile u % tiles,
  // s = u / tiles, and stores its fp32 partial at out + s * split_stride (EPI_STORE32)
  int ksplit, kchunk;
  long split_stride;
  unsigned long long* trace;  // diagnostic timeline (see zo_gemm.h), nullptr in production
  // per-column bias (OPT arch; see zo_gemm.h) and the ReLU activation of EPI_GELU16*
  const float* bias;
  int bias_rps;
  long bias_vstride;
  int relu;
  // EPI_UPDATE64 plans / EPI_UPDATE32 kernel (see zo_gemm.h)
  double* upd_w64;
  void* upd_w16;
  int upd_ld64, upd_ld16, upd_transposed;
  int upd_m32;  // the master holds fp32 values (zo_set_update_mode 1): half the master bytes
  int upd_shadow_rm;  // transposed update whose 16-bit shadow is row-major [i][j] (the embedding)
  int res_tma;  // the epilogue output goes through tmO: the residual as a TMA reduce-add
                // (EPI_RESID32), 16-bit outputs as TMA stores (EPI_STORE16 / GELU16 / GELU16_EXT)
  int relaxed_arrive;  // accumulator hand-back with a relaxed arrive (ZO_RELAXED_ARRIVE=0: release)
  const double* upd_out4;
  double upd_lr, upd_scale;
  const unsigned* upd_abort;
};

// Work segments of one unit: (tile, k-block range).  Data-parallel phase: whole
// tiles unit + i*units below sk_dp (M-fastest order, so the units resident at once
// share weight tiles in L2); stream-K tail (sk = 1): the remaining (< one wave of)
// tiles' k-iterations split evenly, unit u owning [sk_dp*kb + u*sk_w, +sk_w) -- the
// units working on one tile read disjoint k-slices, so no operand is fetched twice.
struct SegIter {
  int cursor, hi, dp, step, unit;
  int hf = 0;  // 0: full tile; 1 / 2: first / second half-width tile of a tail tile
  __device__ __forceinline__ void init(const GemmParams& p, int cg = 1) {
    dp = 1;
    unit = blockIdx.x / cg;  // CTA pairs share one tile (and one stream-K range) when cg = 2
    cursor = unit;
    step = gridDim.x / cg;
    const int tiles = p.m_tiles * p.n_tiles;
    hi = p.sk ? p.sk_dp : p.half_n ? p.half_dp + 2 * (tiles - p.half_dp) : tiles;
    if (p.ksplit) hi = 1;  // one (tile, k-chunk) segment per CTA
  }
  __device__ __forceinline__ bool next(const GemmParams& p, int& tile, int& k0, int& k1) {
    if (p.ksplit) {
      if (cursor >= hi) return false;
      const int tiles = p.m_tiles * p.n_tiles;
      tile = unit % tiles;
      k0 = (unit / tiles) * p.kchunk;
      k1 = min(p.num_kb, k0 + p.kchunk);
      hf = 0;
      cursor = hi;
      return true;
    }
    if (dp) {
      if (cursor < hi) {
        if (p.half_n && cursor >= p.half_dp) {
          const int h = cursor - p.half_dp;
          tile = p.half_dp + (h >> 1);
          hf = 1 + (h & 1);
        } else {
          tile = cursor;
          hf = 0;
        }
        k0 = 0;
        k1 = p.num_kb;
        cursor += step;
        return true;
      }
      if (!p.sk) return false;
      dp = 0;
      const int total = p.m_tiles * p.n_tiles * p.num_kb;
      cursor = p.sk_dp * p.num_kb + unit * p.sk_w;
      hi = min(total, cursor + p.sk_w);
    }
    if (cursor >= hi) return false;
    tile = cursor / p.num_kb;
    k0 = cursor - tile * p.num_kb;
    k1 = min(p.num_kb, hi - tile * p.num_kb);
    cursor = tile * p.num_kb + k1;
    return true;
  }
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// DT: operand type -- 0 fp16, 1 bf16 (kind::f16, 64 elements per 128-byte K block, K = 16
// per MMA), 2 tf32 (kind::tf32 on fp32 storage, 32 elements per K block, K = 8 per MMA; the
// same 32 bytes per MMA step, so the smem ring and descriptors are shared)
template <int BN, int EPI, int DT, int XR, int CG>
__global__ void __launch_bounds__(EPI == EPI_UPDATE32 || EPI == EPI_GELU16 || EPI == EPI_GELU16_EXT ? 320 : 192, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmO, GemmParams p) {
  // EPI_UPDATE32: the tensor update over fp32 masters (the kernel variant of EPI_UPDATE64 plans)
  constexpr bool UPD = EPI == EPI_UPDATE32, M32 = UPD;
  // epilogue warp groups: the update and GELU variants run two groups of 4 warps (320 threads)
  // -- one warp per scheduler leaves their epilogues latency-bound (the update's read-modify-
  // write of every master block; GELU + the extension dot products, ~as long as a d = 2048
  // tile's MMAs).  Update: group g takes the master-block rounds / column chunks = g mod 2;
  // GELU: group g takes the tile's 128-column half g (all of a half-width or <= 128 tile).
  constexpr bool GELU = (EPI == EPI_GELU16 || EPI == EPI_GELU16_EXT);
  constexpr int EGRP = (UPD || GELU) ? 2 : 1;
  // the extension partials t += a . P are summed per 128-column slot (min(BN, 128)): a full
  // tile, its two half-width tail tiles and either epilogue group give the same sums
  constexpr int SLOT = BN < 128 ? BN : 128;
  constexpr bool RES = EPI == EPI_RESID32;
  // TMA-staged epilogue outputs: the residual reduce-add (RES) and the 16-bit stores
  constexpr bool OBOX = RES || EPI == EPI_STORE16 || EPI == EPI_GELU16 || EPI == EPI_GELU16_EXT;
  using C = GemmCfg<BN, CG, UPD, OBOX>;
  constexpr bool BF16 = DT == 1, TF32 = DT == 2;
  constexpr int KE = TF32 ? 32 : 64;  // K elements per 128-byte block
  constexpr uint32_t FMT = TF32 ? 2u : BF16 ? 1u : 0u;  // instruction-descriptor a/b format
  static_assert(!TF32 || EPI == EPI_STORE32 || EPI == EPI_RESID32, "tf32 operands: fp32 epilogues only");
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;  // CTA within the pair
  const bool leader = rank == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sW = smem + C::STAGES * C::STAGE_BYTES;  // EPI_UPDATE32 master-block ring
  uint8_t* sO = sW + C::W_SLOTS * C::W_BYTES;  // OBOX staging boxes (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + C::O_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4 + 2 * C::W_SLOTS);
  // the tensor update (EPI_UPDATE32): fp32 master blocks TMA-loaded through the sW ring
  const bool wtma = UPD && p.upd_transposed;
  const uint32_t wfull0 = smem_u32(bars + 2 * C::STAGES + 4), wempty0 = wfull0 + 8 * C::W_SLOTS;
  // master-block ring geometry: fp32 masters use twice the slots at half the size
  constexpr int wslots = C::W_SLOTS;
  constexpr uint32_t wbytes = C::W_BYTES;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + C::STAGES);
  const uint32_t tfull0 = smem_u32(bars + 2 * C::STAGES), tempty0 = smem_u32(bars + 2 * C::STAGES + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (p.half_n || wtma) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB2)) : "memory");
    if (OBOX && p.res_tma) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmO)) : "memory");
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 4 * EGRP * CG);  // every epilogue warp of the pair arrives at the leader
    }
    for (int w = 0; w < C::W_SLOTS; ++w) {
      mbar_init(wfull0 + 8 * w, 1);
      mbar_init(wempty0 + 8 * w, 4);  // the group's 4 warps release a slot
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done (barriers, TMEM, descriptor prefetch): from here on the operands and
  // the residual are read, so wait for the producing kernel (PDL, zo_common.cuh)
  pdl_wait();
  unsigned long long* tr = p.trace ? p.trace + (size_t)blockIdx.x * 64 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  const int num_tiles = p.m_tiles * p.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int wround = 0;  // EPI_UPDATE32: master blocks issued so far
      SegIter si;
      si.init(p, CG);
      int t, k0, k1;
      while (si.next(p, t, k0, k1)) {
        const int m0 = (t % p.m_tiles) * (C::BM * CG) + (int)rank * C::BM;
        const int hf = si.hf;
        // a half-width tile loads half of the B rows per CTA (tmB2's box)
        const int n0 = hf ? (t / p.m_tiles) * BN + (hf - 1) * (BN / 2) + (int)rank * (BN / 2 / CG)
                          : (t / p.m_tiles) * BN + (int)rank * (BN / CG);
        const CUtensorMap* tb = hf ? &tmB2 : &tmB;
        const uint32_t stage_bytes = hf ? C::A_BYTES + C::B_BYTES / 2 : C::STAGE_BYTES;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t fb = full0 + 8 * stage;
          if constexpr (CG == 2) {
            if (leader) mbar_arrive_expect_tx(fb, 2 * stage_bytes);
            tma_load_2d_cg2(smem_u32(sA + stage * C::A_BYTES), &tmA, fb, (p.kb0 + kb) * KE, m0);
            tma_load_2d_cg2(smem_u32(sB + stage * C::B_BYTES), tb, fb, (p.kb0 + kb) * KE, n0);
          } else {
            mbar_arrive_expect_tx(fb, stage_bytes);
            tma_load_2d(smem_u32(sA + stage * C::A_BYTES), &tmA, fb, (p.kb0 + kb) * KE, m0);
            tma_load_2d(smem_u32(sB + stage * C::B_BYTES), tb, fb, (p.kb0 + kb) * KE, n0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (UPD) {
          // this CTA's master block rows = D columns (input index i), block cols = its 128
          // D rows (output index j); tmB2 is the float64 map over W64 [m, n]
          if (wtma) {
            const int j0 = (t % p.m_tiles) * (C::BM * CG) + (int)rank * C::BM;
            const int i0 = (t / p.m_tiles) * BN;
            for (int r = 0; r < BN / 32; ++r, ++wround) {
              const int ws = wround % wslots;
              mbar_wait(wempty0 + 8 * ws, ((wround / wslots) & 1) ^ 1);
              mbar_arrive_expect_tx(wfull0 + 8 * ws, wbytes);
              tma_load_2d(smem_u32(sW + ws * wbytes), &tmB2, wfull0 + 8 * ws, j0, i0 + 32 * r);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = (1u << 4) | (FMT << 7) | (FMT << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)((C::BM * CG) >> 4) << 24);
      constexpr uint32_t idesc_h = (1u << 4) | (FMT << 7) | (FMT << 10) | ((uint32_t)((BN / 2) >> 3) << 17) |
                                   ((uint32_t)((C::BM * CG) >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      SegIter si;
      si.init(p, CG);
      int t, k0, k1;
      for (; si.next(p, t, k0, k1); ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        if (tr && it < 15) tr[2 + 2 * it] = globaltimer();
        const uint32_t tmem_d = tmem_base + acc * BN;
        const uint32_t id = si.hf ? idesc_h : idesc;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(full0 + 8 * stage, phase);
          tc_fence_after();
          const uint64_t ad = sw128_desc(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bd = sw128_desc(smem_u32(sB + stage * C::B_BYTES));
          const int ks = (kb == p.num_kb - 1) ? p.last_ksteps : 4;
          for (int k = 0; k < ks; ++k) {
            if constexpr (CG == 2)
              tc_mma_cg2<TF32>(tmem_d, ad + 2 * k, bd + 2 * k, id, (kb > k0 || k > 0) ? 1u : 0u);
            else
              tc_mma<TF32>(tmem_d, ad + 2 * k, bd + 2 * k, id, (kb > k0 || k > 0) ? 1u : 0u);
          }
          if constexpr (CG == 2)
            tc_commit_cg2(empty0 + 8 * stage);
          else
            tc_commit(empty0 + 8 * stage);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2)
          tc_commit_cg2(tfull0 + 8 * acc);
        else
          tc_commit(tfull0 + 8 * acc);
        if (tr && it < 15) tr[3 + 2 * it] = globaltimer();
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int grp = (warp - 2) >> 2;  // epilogue warp group (0 unless UPD)
    int wround_e = 0;        // EPI_UPDATE32: master blocks consumed so far (all groups, global order)
    int obuf = 0;            // EPI_RESID32 (TMA path): this warp's staging box to fill next
    const int erow = q * 32 + lane;  // row within the 128-row tile
    int it = 0;
    SegIter si;
    si.init(p, CG);
    int t, k0, k1;
    for (; si.next(p, t, k0, k1); ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (t % p.m_tiles) * (C::BM * CG) + (int)rank * C::BM;
      const int n0 = (t / p.m_tiles) * BN + (si.hf ? (si.hf - 1) * (BN / 2) : 0);
      const int bnc = si.hf ? BN / 2 : BN;  // columns of this (possibly half-width) tile
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      if (tr && warp == 2 && lane == 0 && it < 15) tr[32 + 2 * it] = globaltimer();
      const int row = m0 + erow;
      const bool row_ok = row < p.M;
      if (k0 > 0 && !p.ksplit) {
        // not the tile's first k-block: publish the raw fp32 partial for the owner
        // [BN/4][128 rows] float4 layout: the 32 lanes of a store write 512 contiguous bytes
        float4* ws = reinterpret_cast<float4*>(p.sk_ws + (size_t)blockIdx.x * C::BM * BN) + erow;
#pragma unroll 1
        for (int c = 32 * grp; c < BN; c += 32 * EGRP) {
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            ws[(size_t)(c / 4 + j) * C::BM] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2)
            mbar_arrive_remote(tempty0 + 8 * acc, 0);
          else
            mbar_arrive(tempty0 + 8 * acc);
        }
        __threadfence();
        named_bar_sync(1, 128 * EGRP);
        if (warp == 2 && lane == 0) st_release(p.sk_flags + blockIdx.x, 1u);
        continue;
      }
      // owner (holds the tile's first k-block) of a tile whose later k-blocks were done
      // by units si.unit+1 .. jend-1; their segments are their FIRST tail segments, so
      // no unit's publication waits on another's (no dependency chains)
      int jfirst = si.unit + 1, jend = si.unit + 1;
      if (k1 < p.num_kb && !p.ksplit) jend = ((t + 1) * p.num_kb - 1 - p.sk_dp * p.num_kb) / p.sk_w + 1;
      const bool split = jfirst < jend;
      if (split) {
        // one lane per warp polls (with backoff, so the spinning owners do not hammer the
        // flags' L2 slice while the tail's TMA traffic is in flight); __syncwarp orders
        // the acquire before the other lanes' partial loads
        if (lane == 0)
          for (int j = jfirst; j < jend; ++j)
            for (uint32_t i = 0; ld_acquire(p.sk_flags + j * CG + (int)rank) == 0u; ++i) {
              __nanosleep(128);
              if (i > (1u << 24)) __trap();
            }
        __syncwarp();
      }
      // own accumulator (the tile's first k-blocks) + the partials in ascending k order
      auto add_partials = [&](float (&v)[32], int c) {
        // two partials' chunks in flight per step (16 independent 16-byte loads per lane)
        int j = jfirst;
#pragma unroll 1
        for (; j + 1 < jend; j += 2) {
          const float4* wa =
              reinterpret_cast<const float4*>(p.sk_ws + (size_t)(j * CG + (int)rank) * C::BM * BN) + erow;
          const float4* wb = wa + (size_t)CG * C::BM * BN / 4;
          float4 a[8], b[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            a[e] = wa[(size_t)(c / 4 + e) * C::BM];
            b[e] = wb[(size_t)(c / 4 + e) * C::BM];
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            v[4 * e] = (v[4 * e] + a[e].x) + b[e].x;
            v[4 * e + 1] = (v[4 * e + 1] + a[e].y) + b[e].y;
            v[4 * e + 2] = (v[4 * e + 2] + a[e].z) + b[e].z;
            v[4 * e + 3] = (v[4 * e + 3] + a[e].w) + b[e].w;
          }
        }
        if (j < jend) {
          const float4* wa =
              reinterpret_cast<const float4*>(p.sk_ws + (size_t)(j * CG + (int)rank) * C::BM * BN) + erow;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 w = wa[(size_t)(c / 4 + e) * C::BM];
            v[4 * e] += w.x;
            v[4 * e + 1] += w.y;
            v[4 * e + 2] += w.z;
            v[4 * e + 3] += w.w;
          }
        }
      };
      constexpr bool OUT16 = (EPI == EPI_STORE16 || GELU);
      // this warp's columns of the tile: group g of a GELU kernel its slot g, else all
      const int cb = GELU ? grp * SLOT : 0;
      const int ce = GELU ? (cb + SLOT < bnc ? cb + SLOT : bnc) : bnc;
      float tp[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) tp[k] = 0.f;
      const float* xP = nullptr;
      if constexpr (EPI == EPI_GELU16_EXT) xP = (row < p.xrps) ? p.xPp : p.xPm;
      const float* bb = p.bias ? p.bias + ((row < p.bias_rps) ? 0 : p.bias_vstride) + n0 : nullptr;
      auto add_bias = [&](float (&v)[32], int c) {
        const float4* b4 = reinterpret_cast<const float4*>(bb + c);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 w = __ldg(b4 + j);
          v[4 * j] += w.x;
          v[4 * j + 1] += w.y;
          v[4 * j + 2] += w.z;
          v[4 * j + 3] += w.w;
        }
      };
      if constexpr (M32) {
        if (wtma) {
          // projection, fp32 master W32[i][j] (row i = input, contiguous in the output j):
          // the master block of round r ([32 i][128 j]) arrives by TMA (the ring keeps up to
          // 8 blocks = 128 KB per SM in flight); lane = tile row = output j reads its column,
          // updates it with D[j][i0..i0+31] from its TMEM row and writes it straight back --
          // for a fixed i the 32 lanes store one 128-byte line -- together with its 16-bit
          // shadow row segment W16T[j][i0..i0+31] (64 B).  The slot returns to the producer
          // as soon as the group's 4 warps have read it: no staging of the stores, no
          // barriers between warps.
          const bool skip = p.upd_abort ? (*p.upd_abort != 0u)
                                        : !(isfinite(p.upd_out4[0]) && isfinite(p.upd_out4[1]));
          const float alpha32 = (float)(-(p.upd_lr * p.upd_out4[2]) * p.upd_scale);
          float* W32 = reinterpret_cast<float*>(p.upd_w64);
          const size_t ld = (size_t)p.upd_ld64;
          const int rbase = wround_e;
#pragma unroll 1
          for (int r = grp; r < BN / 32; r += EGRP) {
            const int gi = rbase + r;
            const int ws = gi % wslots;
            float v[32];
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + 32 * r, v);
            mbar_wait(wfull0 + 8 * ws, (gi / wslots) & 1);
            const float* blk32 = reinterpret_cast<const float*>(sW + ws * wbytes) + erow;
            const int col0 = n0 + 32 * r;
            float w[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] = blk32[i * C::BM];
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(wempty0 + 8 * ws);  // this warp is done with the slot
            if (!skip && row_ok) {
              float* dst = W32 + (size_t)col0 * ld + row;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                w[i] = fmaf(alpha32, v[i], w[i]);
                if (col0 + i < p.N) __stcs(dst + (size_t)i * ld, w[i]);
              }
              {
              if (p.upd_shadow_rm) {  // E16[i][j]: for a fixed i the lanes write 64 contiguous bytes
                uint16_t* o = reinterpret_cast<uint16_t*>(p.upd_w16) + (size_t)col0 * p.upd_ld16 + row;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < p.N) o[(size_t)i * p.upd_ld16] = (uint16_t)(pack2<BF16>(w[i], 0.f) & 0xffffu);
              } else {
              uint16_t* o = reinterpret_cast<uint16_t*>(p.upd_w16) + (size_t)row * p.upd_ld16 + col0;
              if (col0 + 32 <= p.N && (((size_t)row * p.upd_ld16 + col0) % 8) == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  uint4 u;
                  u.x = pack2<BF16>(w[8 * j], w[8 * j + 1]);
                  u.y = pack2<BF16>(w[8 * j + 2], w[8 * j + 3]);
                  u.z = pack2<BF16>(w[8 * j + 4], w[8 * j + 5]);
                  u.w = pack2<BF16>(w[8 * j + 6], w[8 * j + 7]);
                  __stcs(reinterpret_cast<uint4*>(o) + j, u);
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < p.N) o[i] = (uint16_t)(pack2<BF16>(w[i], 0.f) & 0xffffu);
              }
              }
              }
            }
          }
          wround_e = rbase + BN / 32;
          goto tile_done;
        }
        __trap();  // update plans are transposed (gemm_set_update_master checks it)
      }
      if constexpr (EPI == EPI_RESID32) {
        if (p.res_tma) {
          // x32 += acc as a TMA reduce-add: each warp stages its 32 rows x 32 columns in a
          // SWIZZLE_128B box (lane = row, 16-byte chunk j at j ^ (row & 7): 4-way banked,
          // the minimum for 512 B) and one lane issues cp.reduce.async.bulk .add.f32 -- the
          // residual read-modify-write happens in L2 (one fp32 round-to-nearest add per
          // element, as before), none of it through the SM's load/store path.  Two boxes per
          // warp alternate; a box is refilled once its previous reduce has read it.  Rows
          // past M and columns past N are clipped by the tensor map.
          uint8_t* box0 = sO + (size_t)(warp - 2) * 2 * 4096;
#pragma unroll 1
          for (int c = 0; c < bnc; c += 32) {
            const int col0 = n0 + c;
            // columns past N (a partial last tile): nothing to add -- and no staging write, which
            // could overwrite the box the last issued reduce is still reading
            if (col0 >= p.N) break;
            float v[32];
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
            if (split) add_partials(v, c);
            if (bb) {
              if (col0 + 32 <= p.N)
                add_bias(v, c);
              else
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < p.N) v[i] += bb[c + i];
            }
            uint8_t* box = box0 + obuf * 4096;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            float4* rowp = reinterpret_cast<float4*>(box + lane * 128);
#pragma unroll
            for (int j = 0; j < 8; ++j) rowp[j ^ (lane & 7)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              asm volatile(
                  "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                      reinterpret_cast<uint64_t>(&tmO)),
                  "r"(col0), "r"(m0 + q * 32), "r"(smem_u32(box))
                  : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            obuf ^= 1;
          }
          goto tile_done;
        }
        // fast path: whole tile row in range -> residual loads for chunk c+1 are in
        // flight while chunk c is added and stored
        const size_t lin0 = (size_t)row * p.ldo + n0;
        // warp-uniform (tcgen05.ld is .sync.aligned)
        if (__all_sync(0xffffffffu, row_ok && n0 + bnc <= p.N && (lin0 % 4) == 0)) {
          float* o = reinterpret_cast<float*>(p.out) + lin0;
          float4 xa[8], xb[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) xa[j] = reinterpret_cast<const float4*>(o)[j];
#pragma unroll 1
          for (int c = 0; c < bnc; c += 32) {
            if (c + 32 < bnc) {
#pragma unroll
              for (int j = 0; j < 8; ++j) xb[j] = reinterpret_cast<const float4*>(o + c + 32)[j];
            }
            float v[32];
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
            if (split) add_partials(v, c);
            if (bb) add_bias(v, c);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4*>(o + c)[j] =
                  make_float4(v[4 * j] + xa[j].x, v[4 * j + 1] + xa[j].y, v[4 * j + 2] + xa[j].z,
                              v[4 * j + 3] + xa[j].w);
#pragma unroll
            for (int j = 0; j < 8; ++j) xa[j] = xb[j];
          }
          goto tile_done;
        }
      }
      if constexpr (OUT16) {
        if (p.res_tma) {
          // 16-bit output through TMA stores: a warp packs 64 columns of its 32 rows into a
          // SWIZZLE_128B box (two 32-column chunks, 16-byte piece j of row r at j ^ (r & 7)) and
          // one lane stores it -- no row-per-lane global stores.  N % 64 == 0 (gemm_plan), so a
          // box is either wholly in range or past N; rows past M are clipped by the map.
          // (one box per warp when two groups share the 32 KB of staging)
          constexpr int NBOX = EGRP == 2 ? 1 : 2;
          uint8_t* box0 = sO + (size_t)(warp - 2) * NBOX * 4096;
#pragma unroll 1
          for (int c = cb; c < ce; c += 32) {
            const int col0 = n0 + c;
            if (col0 >= p.N) break;
            float v[32];
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
            if (split) add_partials(v, c);
            if (bb) add_bias(v, c);
            if constexpr (GELU) {
              if (p.relu) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
              }
            }
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = pack2<BF16>(v[2 * j], v[2 * j + 1]);
            if constexpr (EPI == EPI_GELU16_EXT) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float a = unpack16<BF16>(pk[i >> 1], i & 1);
                if constexpr (XR < 8) {
                  const float* pr = xP + (size_t)(col0 + i) * XR;
#pragma unroll
                  for (int k = 0; k < XR; ++k) tp[k] += a * pr[k];
                } else {
                  const float* pr = xP + (size_t)(col0 + i) * p.xr;
#pragma unroll
                  for (int k = 0; k < 8; ++k)
                    if (k < p.xr) tp[k] += a * pr[k];
                }
              }
            }
            const int half = (c >> 5) & 1;
            uint8_t* box = box0 + (NBOX == 2 ? obuf : 0) * 4096;
            if (half == 0) {
              if (lane == 0) {
                if constexpr (NBOX == 2)
                  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else
                  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              }
              __syncwarp();
            }
            uint4* rowp = reinterpret_cast<uint4*>(box + lane * 128);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              rowp[(half * 4 + j) ^ (lane & 7)] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            if (half == 1) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                        reinterpret_cast<uint64_t>(&tmO)),
                    "r"(col0 - 32), "r"(m0 + q * 32), "r"(smem_u32(box))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              }
              obuf ^= 1;
            }
          }
          goto tile_done;
        }
      }
#pragma unroll 1
      for (int c = cb; c < ce; c += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
        if (split) add_partials(v, c);
        const int col0 = n0 + c;
        if (!row_ok || col0 >= p.N) continue;
        const size_t lin = (size_t)row * p.ldo + col0;
        constexpr int VEC = OUT16 ? 8 : 4;
        const bool full = col0 + 32 <= p.N && (lin % VEC) == 0;
        if (bb) {
          if (col0 + 32 <= p.N)
            add_bias(v, c);
          else
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.N) v[i] += bb[c + i];
        }
        if constexpr (OUT16) {
          if constexpr (GELU) {
            if (p.relu) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = pack2<BF16>(v[2 * j], v[2 * j + 1]);
          if constexpr (EPI == EPI_GELU16_EXT) {
            // t_k += a16[row, col] * P[col, k] on the values the next GEMM reads
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (col0 + i < p.N) {
                const float a = unpack16<BF16>(pk[i >> 1], i & 1);
                if constexpr (XR < 8) {
                  const float* pr = xP + (size_t)(col0 + i) * XR;
#pragma unroll
                  for (int k = 0; k < XR; ++k) tp[k] += a * pr[k];
                } else {
                  const float* pr = xP + (size_t)(col0 + i) * p.xr;
#pragma unroll
                  for (int k = 0; k < 8; ++k)
                    if (k < p.xr) tp[k] += a * pr[k];
                }
              }
            }
          }
          uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + lin;
          if (full) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              reinterpret_cast<uint4*>(o)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.N) o[i] = (uint16_t)(pk[i >> 1] >> (16 * (i & 1)));
          }
        } else {
          float* o = reinterpret_cast<float*>(p.out) + lin +
                     (p.ksplit ? (size_t)(k0 / p.kchunk) * (size_t)p.split_stride : (size_t)0);
          if (full) {
            float4 xr4[8];
            if constexpr (EPI == EPI_RESID32) {
#pragma unroll
              for (int j = 0; j < 8; ++j) xr4[j] = reinterpret_cast<const float4*>(o)[j];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 w = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              if constexpr (EPI == EPI_RESID32) {
                w.x += xr4[j].x;
                w.y += xr4[j].y;
                w.z += xr4[j].z;
                w.w += xr4[j].w;
              }
              reinterpret_cast<float4*>(o)[j] = w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (col0 + i < p.N) {
                if constexpr (EPI == EPI_RESID32)
                  o[i] += v[i];
                else
                  o[i] = v[i];
              }
            }
          }
        }
      }
    tile_done:
      if (tr && warp == 2 && lane == 0 && it < 15) tr[33 + 2 * it] = globaltimer();
      if (split) {
        named_bar_sync(1, 128 * EGRP);
        if (warp == 2 && lane < jend - jfirst)  // re-arm the consumed flags for the next launch
          for (int j = jfirst + lane; j < jend; j += 32) p.sk_flags[j * CG + (int)rank] = 0u;
      }
      if constexpr (EPI == EPI_GELU16_EXT) {
        if (row_ok && cb < ce && n0 + cb < p.N) {
          float* dst = p.tpart + ((size_t)((n0 + cb) / SLOT) * p.tpart_ld + row) * p.xr;
          for (int k = 0; k < p.xr && k < 8; ++k) dst[k] = tp[k];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        // the accumulator hand-back orders only the TMEM reads (tcgen05.fence::before_thread_sync
        // above); the epilogue's global stores need no ordering against the next MMA, so a
        // relaxed arrive -- a release arrive would first wait for them to be acknowledged
        if (p.relaxed_arrive || M32) {
          if constexpr (CG == 2)
            mbar_arrive_remote_relaxed(tempty0 + 8 * acc, 0);
          else
            mbar_arrive_relaxed(tempty0 + 8 * acc);
        } else if constexpr (CG == 2) {
          mbar_arrive_remote(tempty0 + 8 * acc, 0);
        } else {
          mbar_arrive(tempty0 + 8 * acc);
        }
      }
    }
  }
  if constexpr (OBOX)
    if (p.res_tma && warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[1] = globaltimer();
  if constexpr (CG == 2) cluster_sync_all();  // the pair's MMAs/epilogues are done before TMEM is freed
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                   : "memory");
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    ZO_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (!ptr || q != cudaDriverEntryPointSuccess) throw Error(ZO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

void make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                  uint32_t box_rows, int dtype) {
  const bool f32 = dtype == 2;  // tf32 operands on fp32 storage: 32 elements per 128-byte box row
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {f32 ? 32u : 64u, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                     : dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                            const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(ZO_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows=" +
                                 std::to_string(rows) + " cols=" + std::to_string(cols) + " ld=" +
                                 std::to_string(ld));
}

void gemm_set_update_master(GemmDesc& g) {
  // EPI_UPDATE64 plan (run by the EPI_UPDATE32 kernel): an fp32 map over the master
  // W[N (inputs), M (outputs)] (row stride upd_ld64), 32 x 128 boxes, no swizzle -- streamed
  // through the kernel's master-block ring in place of the half-tile B map
  if (g.epi != EPI_UPDATE64) return;
  if (!g.upd_m32 || !g.upd_transposed)
    throw Error(ZO_ERR_INTERNAL, "tensor update: fp32 master, transposed plan (D = V U^T) only");
  if (g.cg != 1 && g.cg != 2) throw Error(ZO_ERR_INTERNAL, "bad CTA group");
  if (g.bn % 32 || g.half_n || g.sk) throw Error(ZO_ERR_INTERNAL, "update GEMM: plain tiles only");
  cuuint64_t dims[2] = {(cuuint64_t)g.M, (cuuint64_t)g.N};
  cuuint64_t strides[1] = {(cuuint64_t)g.upd_ld64 * 4};
  cuuint32_t box[2] = {128, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&g.tmB2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                            g.upd_w64, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(ZO_ERR_CUDA, "cuTensorMapEncodeTiled (float64 master) failed");
}

void gemm_plan(GemmDesc& g, const void* A, int M, int lda, const void* B, int N, int ldb, int Kp_used, int epi,
               int dtype, void* out, int ldo, int num_sms, int bn_hint) {
  if (lda % 8 || ldb % 8) throw Error(ZO_ERR_DIMENSION, "GEMM leading dimensions must be multiples of 8");
  if (dtype == 2 && epi != EPI_STORE32 && epi != EPI_RESID32)
    throw Error(ZO_ERR_INTERNAL, "tf32 GEMM supports the fp32 epilogues only");
  g.M = M;
  g.N = N;
  g.epi = epi;
  g.bf16 = dtype;
  g.out = out;
  g.ldo = ldo;
  const int ke = dtype == 2 ? 32 : 64;  // K elements per 128-byte block
  g.num_kb = (Kp_used + ke - 1) / ke;
  const int rem = Kp_used - ke * (g.num_kb - 1);
  g.last_ksteps = (rem + ke / 4 - 1) / (ke / 4);
  const int m_tiles = (M + 127) / 128;
  // tile N: prefer 256 unless that leaves the GPU badly under-filled
  int bn = 256;
  if (N <= 64)
    bn = 64;
  else if (N <= 128 || (int64_t)m_tiles * ((N + 255) / 256) < num_sms / 2)
    bn = (int64_t)m_tiles * ((N + 127) / 128) < num_sms / 2 ? 64 : 128;  // small M: spread the weight read
  if (bn_hint) bn = bn_hint;  // the caller knows better (split-K skinny GEMMs: one N tile reads A once)
  g.bn = bn;
  // CTA pairs (M = 256 per tile) halve the per-CTA B traffic and double the stages
  static const bool cg2_on = [] {
    const char* e = std::getenv("ZO_CG2");
    return !e || std::atoi(e) != 0;
  }();
  g.cg = (cg2_on && N > 128 && bn >= 128 && M >= 512) ? 2 : 1;
  // the update kernel's master-block ring leaves no room for 256-wide single-CTA operand tiles
  if (epi == EPI_UPDATE64 && g.cg == 1 && bn > 128) g.bn = bn = 128;
  // N=128 pair tiles measured 1.4-1.5x slower (A re-reads, fixed costs), 192-wide no
  // faster than 256 on the ragged 13B shapes (they re-read A 33% more)
  if (g.cg == 2) g.bn = bn = 256;
  const int mt = (M + 128 * g.cg - 1) / (128 * g.cg);
  const int tiles = mt * ((N + bn - 1) / bn);
  const int slots = num_sms / g.cg;
  g.grid = (tiles < slots ? tiles : slots) * g.cg;
  const int mrows = ((M + 127) / 128) * 128;
  make_tmap_2d(&g.tmA, A, (uint64_t)mrows, (uint64_t)lda, (uint64_t)lda, 128, dtype);
  make_tmap_2d(&g.tmB, B, (uint64_t)N, (uint64_t)ldb, (uint64_t)ldb, (uint32_t)(bn / g.cg), dtype);
  make_tmap_2d(&g.tmB2, B, (uint64_t)N, (uint64_t)ldb, (uint64_t)ldb, (uint32_t)(bn / g.cg / 2), dtype);
  g.half_dp = g.half_n = 0;
  // EPI_RESID32: the residual x32[M, N] (row stride ldo) as a TMA reduce-add target, 32 x 32
  // fp32 boxes, SWIZZLE_128B (ZO_RES_TMA=0 keeps the load/add/store epilogue)
  static const bool res_tma_on = [] {
    const char* e = std::getenv("ZO_RES_TMA");
    return !e || std::atoi(e) != 0;
  }();
  g.res_tma = 0;
  static const bool out_tma_on = [] {
    const char* e = std::getenv("ZO_OUT_TMA");
    return !e || std::atoi(e) != 0;
  }();
  const bool out16 = epi == EPI_STORE16 || epi == EPI_GELU16 || epi == EPI_GELU16_EXT;
  if (out16 && dtype != 2 && out_tma_on && N % 64 == 0 && ((size_t)ldo * 2) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(out) % 16) == 0) {
    // 16-bit outputs through TMA stores: [M, N] (row stride ldo) in 32 x 64 boxes, SWIZZLE_128B
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)ldo * 2};
    cuuint32_t box[2] = {64, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&g.tmO, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, out, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(ZO_ERR_CUDA, "cuTensorMapEncodeTiled (16-bit output) failed");
    g.res_tma = 1;
  }
  if (epi == EPI_RESID32 && res_tma_on && ((size_t)ldo * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(out) % 16) == 0) {
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)ldo * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&g.tmO, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(ZO_ERR_CUDA, "cuTensorMapEncodeTiled (residual) failed");
    g.res_tma = 1;
  }
}

static int max_pair_units(int num_sms);

void gemm_enable_halftail(GemmDesc& g, int num_sms) {
  // pair tiles only, no stream-K (the GELU epilogue's extension partials are per 128-column
  // slot, so half-width tiles write whole slots)
  static const bool on = [] {
    const char* e = std::getenv("ZO_HALFTAIL");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || g.sk || g.cg != 2 || g.bn != 256) return;
  int units = std::min(g.grid / 2, max_pair_units(num_sms));
  const int m_tiles = (g.M + 255) / 256, n_tiles = (g.N + 255) / 256;
  const int tiles = m_tiles * n_tiles;
  if (units < 2 || tiles <= units || tiles % units == 0) return;
  const int tail = tiles % units;
  // the last wave's 2*tail half tiles must still fit one round
  if (2 * tail > units) return;
  g.half_dp = tiles - tail;
  g.half_n = 1;
  g.grid = units * 2;
}

template <int BN, int EPI, int BF16, int XR, int CG>
static void launch_t(const GemmDesc& g, cudaStream_t st, int kb0 = 0, int nkb = -1, int last_ksteps = -1) {
  using C = GemmCfg<BN, CG, EPI == EPI_UPDATE32,
                    EPI == EPI_RESID32 || EPI == EPI_STORE16 || EPI == EPI_GELU16 || EPI == EPI_GELU16_EXT>;
  constexpr int NT = (EPI == EPI_UPDATE32 || EPI == EPI_GELU16 || EPI == EPI_GELU16_EXT) ? 320 : 192;  // k_gemm's launch bounds
  static bool attr_set = false;
  if (!attr_set) {
    ZO_CUDA_TRY(cudaFuncSetAttribute(k_gemm<BN, EPI, BF16, XR, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::SMEM));
    attr_set = true;
  }
  GemmParams p;
  p.M = g.M;
  p.N = g.N;
  p.kb0 = kb0;
  p.num_kb = nkb < 0 ? g.num_kb : nkb;
  p.last_ksteps = last_ksteps < 0 ? g.last_ksteps : last_ksteps;
  p.m_tiles = (g.M + 128 * CG - 1) / (128 * CG);
  p.n_tiles = (g.N + BN - 1) / BN;
  p.ldo = g.ldo;
  p.out = g.out;
  p.xPp = g.xPp;
  p.xPm = g.xPm;
  p.xr = g.xr;
  p.xrps = g.xrps;
  p.tpart_ld = g.tpart_ld;
  p.tpart = g.tpart;
  p.sk = g.sk;
  p.sk_w = g.sk_w;
  p.sk_dp = g.sk_dp;
  p.sk_ws = g.sk_ws;
  p.sk_flags = g.sk_flags;
  p.half_dp = g.half_dp;
  p.trace = g.trace;
  p.half_n = g.half_n;
  p.bias = kb0 == 0 ? g.bias : nullptr;  // a K-chunked launch adds the bias once
  p.bias_rps = g.bias_rps;
  p.bias_vstride = g.bias_vstride;
  p.relu = g.relu;
  p.ksplit = g.ksplit;
  p.kchunk = g.kchunk;
  p.split_stride = g.split_stride;
  p.upd_w64 = g.upd_w64;
  p.upd_w16 = g.upd_w16;
  p.upd_ld64 = g.upd_ld64;
  p.upd_ld16 = g.upd_ld16;
  p.upd_transposed = g.upd_transposed;
  p.upd_m32 = g.upd_m32;
  p.upd_shadow_rm = g.upd_shadow_rm;
  p.res_tma = g.res_tma;
  {
    static const int relaxed = [] {
      const char* e = std::getenv("ZO_RELAXED_ARRIVE");
      return (!e || std::atoi(e) != 0) ? 1 : 0;
    }();
    p.relaxed_arrive = relaxed;
  }
  p.upd_out4 = g.upd_out4;
  p.upd_lr = g.upd_lr;
  p.upd_scale = g.upd_scale;
  p.upd_abort = g.upd_abort;
  if constexpr (CG == 1) {
    launch_pdl(k_gemm<BN, EPI, BF16, XR, 1>, dim3(g.grid), dim3(NT), C::SMEM, st, g.tmA, g.tmB, g.tmB2, g.tmO, p);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    ZO_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_gemm<BN, EPI, BF16, XR, 2>, g.tmA, g.tmB, g.tmB2, g.tmO, p));
  }
}

// tf32 operands (the real32 path's 3xTF32 GEMMs).  The tensor core's fp32 accumulation
// truncates on every MMA, an error growing linearly with the number of accumulations
// (measured: ~1e-8 x K relative, scripts/diag_tf32.py), so K is cut into chunks of
// ZO_TF32_KCHUNK 32-wide blocks (default 4 = 16 MMAs; K = 4096: 4e-5 unchunked, 2.9e-6 at 8,
// 1.9e-6 at 4 -- fp32-GEMM class): the first chunk stores (or adds
// into the residual), every later chunk adds its fp32 partial with a round-to-nearest
// add in the epilogue (EPI_RESID32).
static int tf32_kchunk() {
  static const int kc = [] {
    const char* e = std::getenv("ZO_TF32_KCHUNK");
    const int v = e ? std::atoi(e) : 4;
    return v > 0 ? v : 4;
  }();
  return kc;
}
template <int BN, int CG>
static void launch_e32(const GemmDesc& g, cudaStream_t st) {
  const int kc = tf32_kchunk();
  for (int kb0 = 0; kb0 < g.num_kb; kb0 += kc) {
    const int n = std::min(kc, g.num_kb - kb0);
    const int ls = (kb0 + n == g.num_kb) ? g.last_ksteps : 4;
    if (g.epi == EPI_RESID32 || kb0 > 0) launch_t<BN, EPI_RESID32, 2, 0, CG>(g, st, kb0, n, ls);
    else launch_t<BN, EPI_STORE32, 2, 0, CG>(g, st, kb0, n, ls);
  }
}

template <int BN, bool BF16, int CG>
static void launch_e(const GemmDesc& g, cudaStream_t st) {
  switch (g.epi) {
    case EPI_STORE16: launch_t<BN, EPI_STORE16, BF16, 0, CG>(g, st); break;
    case EPI_GELU16: launch_t<BN, EPI_GELU16, BF16, 0, CG>(g, st); break;
    case EPI_GELU16_EXT:
      if (g.xr == 1) launch_t<BN, EPI_GELU16_EXT, BF16, 1, CG>(g, st);
      else if (g.xr == 2) launch_t<BN, EPI_GELU16_EXT, BF16, 2, CG>(g, st);
      else if (g.xr == 4) launch_t<BN, EPI_GELU16_EXT, BF16, 4, CG>(g, st);
      else launch_t<BN, EPI_GELU16_EXT, BF16, 8, CG>(g, st);
      break;
    case EPI_RESID32: launch_t<BN, EPI_RESID32, BF16, 0, CG>(g, st); break;
    case EPI_UPDATE64:  // fp32 master, transposed (gemm_set_update_master checked both)
      launch_t<BN, EPI_UPDATE32, BF16, 0, CG>(g, st);
      break;
    default: launch_t<BN, EPI_STORE32, BF16, 0, CG>(g, st); break;
  }
}

// Co-resident 2-CTA clusters of the pair kernel (stream-K spins on peers, so every
// unit must be resident at once; a GPC with an odd SM count leaves one SM unpaired).
static int max_pair_units(int num_sms) {
  static int units = -1;
  if (units < 0) {
    using C = GemmCfg<256, 2>;
    auto* fn = k_gemm<256, EPI_STORE16, 0, 0, 2>;
    ZO_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (num_sms / 2));
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = C::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    ZO_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, fn, &cfg));
    units = n;
    if (std::getenv("ZO_DEBUG")) fprintf(stderr, "[zob200] max co-resident CTA pairs: %d\n", n);
  }
  return units;
}

void gemm_enable_streamk(GemmDesc& g, float* ws, unsigned* flags, int num_sms) {
  // Data-parallel whole tiles for every full wave, then the last partial wave's tiles
  // split k-wise over ALL persistent units (CTAs, or CTA pairs when cg = 2), so the
  // ragged last wave disappears.  The units sharing a tail tile read disjoint k-slices
  // of its operands (no re-reads); a full-waves-only (non-tail) stream-K split was
  // measured slower -- units at scattered k offsets lose the L2 sharing of the
  // lock-step data-parallel waves.
  if (!ws || !flags) return;
  const int cg = g.cg;
  int units = g.grid / cg;
  if (cg == 2) units = std::min(units, max_pair_units(num_sms));
  const int m_tiles = (g.M + 128 * cg - 1) / (128 * cg), n_tiles = (g.N + g.bn - 1) / g.bn;
  const int tiles = m_tiles * n_tiles;
  if (units < 2 || tiles <= units || tiles % units == 0) return;
  const int dp_waves = tiles / units;
  const int tail = tiles - dp_waves * units;
  const long sk_iters = (long)tail * g.num_kb;
  int w = (int)((sk_iters + units - 1) / units);
  // too fine: each owner would sum many partials; measured a loss at M=2048 attn_out
  // (12 tail tiles x 81 k-blocks over 74 pairs -> 14 per unit), a gain for ff_down (53)
  // -- except a 4-way split of a small tail (<= units / 4 tail tiles, >= 16 k-blocks per
  // unit): 13B attn_out, 12 tail tiles x 81 k-blocks, 92 -> 87 us (vs half-width tail tiles)
  const bool four_way = 4 * tail <= units && (g.num_kb + 3) / 4 >= 16;
  if (w < 32 && !four_way) return;
  // only a mostly-empty last wave pays for the fixup (13B: ff_down's 12 of 74 pairs,
  // 382 -> 350 us; qkv's 36/74 and ff_up's 48/74 measured neutral-to-worse)
  if (3 * tail > units) return;
  // at most 4 units per tail tile: the owner then sums <= 3 partials (13B ff_down: 6 -> 4
  // participants, 271 -> 265 us); the other units idle through the tail
  if (4 * tail <= units) w = std::max(w, (g.num_kb + 3) / 4);
  g.sk = 1;
  g.sk_dp = dp_waves * units;
  g.sk_w = w;
  g.sk_ws = ws;
  g.sk_flags = flags;
  g.grid = units * cg;
}

int gemm_enable_splitk(GemmDesc& g, int splits, long split_stride) {
  if (g.cg != 1 || g.epi != EPI_STORE32 || g.bf16 == 2) throw Error(ZO_ERR_INTERNAL, "split-K: fp32 single-CTA tiles only");
  const int kc = std::max(1, (g.num_kb + splits - 1) / splits);
  const int s = (g.num_kb + kc - 1) / kc;
  const int tiles = ((g.M + 127) / 128) * ((g.N + g.bn - 1) / g.bn);
  g.ksplit = s;
  g.kchunk = kc;
  g.split_stride = split_stride;
  g.grid = tiles * s;
  g.sk = 0;
  g.half_n = 0;
  return s;
}

void gemm_launch(const GemmDesc& g, cudaStream_t st) {
  if (g.bf16 == 2) {
    if (g.cg == 2) launch_e32<256, 2>(g, st);
    else if (g.bn == 256) launch_e32<256, 1>(g, st);
    else if (g.bn == 128) launch_e32<128, 1>(g, st);
    else launch_e32<64, 1>(g, st);
    return;
  }
  if (g.cg == 2) {
    if (g.bf16) launch_e<256, true, 2>(g, st);
    else launch_e<256, false, 2>(g, st);
    return;
  }
  if (g.bf16) {
    if (g.bn == 256) launch_e<256, true, 1>(g, st);
    else if (g.bn == 128) launch_e<128, true, 1>(g, st);
    else launch_e<64, true, 1>(g, st);
  } else {
    if (g.bn == 256) launch_e<256, false, 1>(g, st);
    else if (g.bn == 128) launch_e<128, false, 1>(g, st);
    else launch_e<64, false, 1>(g, st);
  }
}

}  // namespace zo
