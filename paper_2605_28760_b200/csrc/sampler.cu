// K1 -- bit-exact direction sampler.
//
// Reproduces StreamKey(seed, step, layer_id, role).generator().standard_normal
// (numerics.py:139-168) on the GPU:
//   key   = SeedSequence([seed, step, fnv1a64(layer_id), role]).generate_state(2, u64)
//   u64 p = Philox4x64-10(key, counter = p/4 + 1)[p % 4]
//   x     = numpy's 256-layer ziggurat over those u64s, row-major fill.
//
// The ziggurat consumes a data-dependent number of u64s per sample, so sample i
// cannot be addressed directly.  We parse in parallel with a speculative
// chunk splice:
//   k_spec : every chunk of CH u64 positions is parsed as if an attempt started
//            at its first position -> speculative exit (first attempt start at
//            or past the chunk end), sample count, and which of the chunk's
//            first 8 positions start an attempt / yield a sample.
//   k_scan : one CTA per stream.  Chunk c's true entry is chunk c-1's exit
//            (a few positions into c at most).  When that entry is one of the
//            speculative attempt starts the two parses are the same chain from
//            there on: the true count is the speculative
//            count minus the samples of the skipped attempts, the exit is the
//            speculative exit -- no second Philox pass.  Otherwise (~2e-4 of
//            chunks) the chunk is re-parsed from its entry; a re-parse whose exit
//            differs breaks the splice and the rest of the stream is repaired
//            serially (never observed; counted).  Then counts -> offsets.
//   k_emit : re-parse from the verified entry and write samples in place -- or, with a
//            scratch (SamplerPlan::d_scratch, the direction plans), k_emit_copy: k_spec
//            kept each chunk's speculative samples, and a warp per chunk copies them
//            (minus the d_skip leading ones) to their offsets, coalesced, writing the
//            optional 16-bit / fp32 copies in the same pass; only chunks whose entry fell
//            inside a speculative attempt are re-parsed.
// Philox runs twice per sample without a scratch, once with; every step is exact.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "zo_common.cuh"
#include "zo_glibc_math.cuh"
#include "zo_sampler.h"

#define ZO_ZIG_QUAL __device__ const
#include "ziggurat_tables.h"
#undef ZO_ZIG_QUAL

namespace zo {

static constexpr uint64_t CH = 128;  // u64 positions per chunk

// ---------------------------------------------------------------- SeedSequence
__host__ __device__ inline uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931e8875u;
  v *= hc;
  v ^= v >> 16;
  return v;
}
__host__ __device__ inline uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  return r ^ (r >> 16);
}
__host__ __device__ inline int ss_words(uint64_t v, uint32_t* out) {
  int n = 0;
  if (v == 0) {
    out[n++] = 0;
    return n;
  }
  while (v) {
    out[n++] = (uint32_t)(v & 0xffffffffu);
    v >>= 32;
  }
  return n;
}
// numpy bit_generator.pyx SeedSequence(entropy).generate_state(2, uint64)
__host__ __device__ inline void seed_sequence_key(uint64_t seed, uint64_t step, uint64_t lid_hash,
                                                  uint64_t role, uint64_t key[2]) {
  uint32_t ent[8];
  int n = 0;
  n += ss_words(seed, ent + n);
  n += ss_words(step, ent + n);
  n += ss_words(lid_hash, ent + n);
  n += ss_words(role, ent + n);
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
  uint32_t w[4];
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  key[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  key[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

void host_stream_key(uint64_t seed, uint64_t step, uint64_t lid_hash, uint64_t role, uint64_t key[2]) {
  seed_sequence_key(seed, step, lid_hash, role, key);
}

// ---------------------------------------------------------------- Philox4x64-10
__device__ __forceinline__ void philox_block(uint64_t k0, uint64_t k1, uint64_t blk, uint64_t out[4]) {
  uint64_t c0 = blk + 1, c1 = (c0 == 0) ? 1 : 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

struct Zig {
  const uint64_t* ki;
  const double* wi;
  const double* fi;
};

struct Parser {
  uint64_t k0, k1, pos, blk;
  uint64_t buf[4];
  __device__ void init(uint64_t a, uint64_t b, uint64_t p) {
    k0 = a;
    k1 = b;
    pos = p;
    blk = ~0ULL;
  }
  __device__ __forceinline__ uint64_t next() {
    uint64_t b = pos >> 2;
    if (b != blk) {
      philox_block(k0, k1, b, buf);
      blk = b;
    }
    uint64_t v = buf[pos & 3];
    ++pos;
    return v;
  }
  __device__ __forceinline__ double next_double() {
    return __dmul_rn((double)(next() >> 11), 1.0 / 9007199254740992.0);
  }
  // One attempt of numpy's random_standard_normal outer loop.  Returns true and
  // sets *x when the attempt produced a sample.  *amb counts exp() decisions
  // too close to call between CUDA's exp and glibc's (|lhs-e| <= 2 ulp).
  __device__ __forceinline__ bool attempt(const Zig& z, double* x, unsigned* amb) {
    uint64_t r = next();
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double v = __dmul_rn((double)rabs, z.wi[idx]);
    if (sign) v = -v;
    if (rabs < z.ki[idx]) {
      *x = v;
      return true;
    }
    if (idx == 0) {
      const double R = 3.6541528853610088, INV_R = 0.27366123732975828;
      for (;;) {
        double xx = __dmul_rn(-INV_R, glibc_log1p(-next_double()));
        double yy = -glibc_log1p(-next_double());
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          *x = ((rabs >> 8) & 1) ? -__dadd_rn(R, xx) : __dadd_rn(R, xx);
          return true;
        }
      }
    }
    double u = next_double();
    double lhs = __dadd_rn(__dmul_rn(__dsub_rn(z.fi[idx - 1], z.fi[idx]), u), z.fi[idx]);
    double e = exp(__dmul_rn(__dmul_rn(-0.5, v), v));
    if (fabs(__dsub_rn(lhs, e)) <= __dmul_rn(e, 4.5e-16)) ++*amb;
    if (lhs < e) {
      *x = v;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ void load_tables(Zig& z, uint64_t* ki, double* wi, double* fi) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    ki[i] = zo_zig_ki[i];
    wi[i] = zo_zig_wi[i];
    fi[i] = zo_zig_fi[i];
  }
  __syncthreads();
  z.ki = ki;
  z.wi = wi;
  z.fi = fi;
}

__device__ __forceinline__ uint64_t key_step(const StreamDesc& s, const uint64_t* d_step, uint32_t nu) {
  if (s.step_mode == STEP_FIXED) return s.fixed_step;
  uint64_t t = *d_step;
  if (s.step_mode == STEP_WINDOW) return (t / nu) * nu;
  return t;
}

__global__ void k_keys(const StreamDesc* __restrict__ streams, int S, uint64_t seed,
                       const uint64_t* __restrict__ d_step, uint32_t nu, uint64_t* __restrict__ keys) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  StreamDesc d = streams[s];
  uint64_t k[2];
  seed_sequence_key(d.seed_override ? d.seed_value : seed, key_step(d, d_step, nu), d.lid_hash, d.role, k);
  keys[2 * s] = k[0];
  keys[2 * s + 1] = k[1];
}

__global__ void __launch_bounds__(256) k_spec(const StreamDesc* __restrict__ streams,
                                              const uint32_t* __restrict__ chunk_stream, int64_t C,
                                              const uint64_t* __restrict__ keys,
                                              uint64_t* __restrict__ spec_exit, uint32_t* __restrict__ count,
                                              double* __restrict__ scratch, unsigned* flags) {
  __shared__ uint64_t ki[256];
  __shared__ double wi[256], fi[256];
  Zig z;
  load_tables(z, ki, wi, fi);
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  uint32_t s = chunk_stream[c];
  uint64_t local = (uint64_t)(c - (int64_t)streams[s].chunk_begin);
  uint64_t beg = local * CH, end = beg + CH;
  Parser p;
  p.init(keys[2 * s], keys[2 * s + 1], beg);
  unsigned amb = 0, n = 0, starts = 0, yields = 0;
  double x;
  double* sc = scratch ? scratch + (size_t)c * CH : nullptr;
  while (p.pos < end) {
    const uint64_t at = p.pos - beg;
    const bool y = p.attempt(z, &x, &amb);
    if (y && sc) sc[n] = x;  // raw (unscaled) speculative sample n of the chunk
    n += y ? 1u : 0u;
    if (at < 8) {
      starts |= 1u << at;
      yields |= (y ? 1u : 0u) << at;
    }
  }
  spec_exit[c] = p.pos;
  count[c] = n | (starts << 16) | (yields << 24);
}

// One CTA per stream: verify/repair the splice, exclusive-scan the counts.
__global__ void __launch_bounds__(1024) k_scan(const StreamDesc* __restrict__ streams,
                                               const uint64_t* __restrict__ keys,
                                               const uint64_t* __restrict__ spec_exit,
                                               uint64_t* __restrict__ exit_pos, uint32_t* __restrict__ count,
                                               uint64_t* __restrict__ offset, uint32_t* __restrict__ skip,
                                               unsigned* flags) {
  __shared__ uint64_t ki[256];
  __shared__ double wi[256], fi[256];
  __shared__ int64_t first_bad;
  __shared__ uint64_t warp_sums[32];
  __shared__ uint64_t carry;
  Zig z;
  load_tables(z, ki, wi, fi);
  const StreamDesc d = streams[blockIdx.x];
  const int64_t cb = (int64_t)d.chunk_begin, nc = (int64_t)d.n_chunks;
  if (threadIdx.x == 0) first_bad = nc;
  __syncthreads();
  // true entry of chunk i = exit of chunk i-1 (= its speculative exit unless a re-parse
  // below changed it, which breaks the splice at i+1 and sends the rest to the repair)
  for (int64_t i = threadIdx.x; i < nc; i += blockDim.x) {
    const uint32_t raw = count[cb + i];
    uint32_t n = raw & 0xffffu;
    uint64_t ex = spec_exit[cb + i];
    uint32_t sk = 0;  // leading speculative samples the true parse drops (~0u: re-parse in emit)
    if (i > 0) {
      const uint64_t off = spec_exit[cb + i - 1] - (uint64_t)i * CH;
      const uint32_t starts = (raw >> 16) & 0xffu, yields = raw >> 24;
      if (off < 8 && ((starts >> off) & 1u)) {
        sk = (uint32_t)__popc(yields & ((1u << off) - 1u));
        n -= sk;
      } else {  // the entry falls inside a speculative attempt: re-parse this chunk
        sk = ~0u;
        Parser p;
        p.init(keys[2 * blockIdx.x], keys[2 * blockIdx.x + 1], spec_exit[cb + i - 1]);
        const uint64_t end = (uint64_t)(i + 1) * CH;
        unsigned amb = 0;
        double x;
        n = 0;
        while (p.pos < end) n += p.attempt(z, &x, &amb) ? 1u : 0u;
        if (p.pos != ex) atomicMin((unsigned long long*)&first_bad, (unsigned long long)(i + 1));
        ex = p.pos;
      }
    }
    count[cb + i] = n;
    exit_pos[cb + i] = ex;
    if (skip) skip[cb + i] = sk;
  }
  __syncthreads();
  if (first_bad < nc && threadIdx.x == 0) {
    // serial repair (vanishingly rare): re-parse every chunk after the break
    atomicAdd(&flags[2], 1u);
    unsigned amb = 0;
    double x;
    for (int64_t i = first_bad; i < nc; ++i) {
      Parser p;
      p.init(keys[2 * blockIdx.x], keys[2 * blockIdx.x + 1], exit_pos[cb + i - 1]);
      uint64_t end = (uint64_t)(i + 1) * CH;
      unsigned n = 0;
      while (p.pos < end) n += p.attempt(z, &x, &amb) ? 1u : 0u;
      exit_pos[cb + i] = p.pos;
      count[cb + i] = n;
      if (skip) skip[cb + i] = ~0u;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < nc; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    uint64_t v = i < nc ? count[cb + i] : 0;
    uint64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      uint64_t wi2 = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint64_t t = __shfl_up_sync(0xffffffffu, wi2, o);
        if (lane >= o) wi2 += t;
      }
      warp_sums[lane] = wi2 - w;  // exclusive warp prefix
    }
    __syncthreads();
    uint64_t excl = carry + warp_sums[warp] + incl - v;
    if (i < nc) offset[cb + i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0 && carry < d.n) atomicAdd(&flags[0], 1u);
}

__global__ void __launch_bounds__(256) k_emit(const StreamDesc* __restrict__ streams,
                                              const uint32_t* __restrict__ chunk_stream, int64_t C,
                                              const uint64_t* __restrict__ keys,
                                              const uint64_t* __restrict__ exit_pos,
                                              const uint64_t* __restrict__ offset, double* __restrict__ out,
                                              unsigned* flags) {
  __shared__ uint64_t ki[256];
  __shared__ double wi[256], fi[256];
  Zig z;
  load_tables(z, ki, wi, fi);
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  uint32_t s = chunk_stream[c];
  const StreamDesc& d = streams[s];
  uint64_t local = (uint64_t)(c - (int64_t)d.chunk_begin);
  uint64_t end = (local + 1) * CH;
  uint64_t entry = local == 0 ? 0 : exit_pos[c - 1];
  uint64_t o = offset[c];
  if (o >= d.n) return;
  Parser p;
  p.init(keys[2 * s], keys[2 * s + 1], entry);
  unsigned amb = 0;
  double x;
  double* dst = out + d.out_off;
  const double scale = d.scale;
  const bool scaled = d.apply_scale != 0;
  while (p.pos < end && o < d.n) {
    if (p.attempt(z, &x, &amb)) dst[o++] = scaled ? __dmul_rn(scale, x) : x;
  }
  if (amb) atomicAdd(&flags[1], amb);
}

// store one emitted sample (scaled if the stream asks) and its optional 16-bit / fp32 copies
__device__ __forceinline__ void put_sample(double* dst, uint16_t* d16, bool bf16, float* d32, uint64_t o, double v) {
  dst[o] = v;
  if (d16) {
    const float f = (float)v;
    d16[o] = bf16 ? __bfloat16_as_ushort(__float2bfloat16_rn(f)) : __half_as_ushort(__float2half_rn(f));
  }
  if (d32) d32[o] = (float)v;
}

// Copy emit: a warp takes 32 consecutive chunks at a time -- lane l loads chunk l's metadata
// (stream, offset, skip, count) so the dependent loads are paid once per 32 chunks -- then
// copies each chunk's speculative samples [skip, skip + count) with all 32 lanes (coalesced),
// writing the optional 16-bit / fp32 copies in the same pass.  A chunk whose entry fell
// inside a speculative attempt (skip == ~0u, rare) is re-parsed by its own lane afterwards,
// with the ziggurat tables read from global memory.
__global__ void __launch_bounds__(256) k_emit_copy(const StreamDesc* __restrict__ streams,
                                                   const uint32_t* __restrict__ chunk_stream, int64_t C,
                                                   const uint64_t* __restrict__ keys,
                                                   const uint64_t* __restrict__ exit_pos,
                                                   const uint64_t* __restrict__ offset,
                                                   const uint32_t* __restrict__ count,
                                                   const uint32_t* __restrict__ skip,
                                                   const double* __restrict__ scratch, double* __restrict__ out,
                                                   uint16_t* __restrict__ out16, bool bf16, float* __restrict__ out32,
                                                   int G, unsigned* flags) {
  const Zig z{zo_zig_ki, zo_zig_wi, zo_zig_fi};
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G; c0 < C; c0 += warps * G) {
    // lane-owned metadata of chunk c0 + lane (lanes < G)
    const int64_t c = lane < G ? c0 + lane : C;
    uint64_t o = ~0ull, dn = 0, doff = 0;
    uint32_t sk = 0, cnt = 0, s = 0;
    double scale = 1.0;
    int scaled = 0;
    if (c < C) {
      s = chunk_stream[c];
      const StreamDesc& d = streams[s];
      o = offset[c];
      dn = d.n;
      doff = d.out_off;
      scale = d.scale;
      scaled = d.apply_scale != 0;
      sk = skip[c];
      cnt = count[c];
    }
    const int nj = (int)min((int64_t)G, C - c0);
    for (int j = 0; j < nj; ++j) {
      const uint64_t oj = __shfl_sync(0xffffffffu, o, j);
      const uint64_t dnj = __shfl_sync(0xffffffffu, dn, j);
      const uint32_t skj = __shfl_sync(0xffffffffu, sk, j);
      if (oj >= dnj || skj == ~0u) continue;  // past the stream's end / re-parsed below
      const uint64_t doffj = __shfl_sync(0xffffffffu, doff, j);
      const double scj = __shfl_sync(0xffffffffu, scale, j);
      const int sdj = __shfl_sync(0xffffffffu, scaled, j);
      const uint64_t n = min((uint64_t)__shfl_sync(0xffffffffu, cnt, j), dnj - oj);
      const double* src = scratch + (size_t)(c0 + j) * CH + skj;
      double* dst = out + doffj;
      uint16_t* d16 = out16 ? out16 + doffj : nullptr;
      float* d32 = out32 ? out32 + doffj : nullptr;
#pragma unroll 4
      for (uint64_t i = lane; i < n; i += 32) {
        const double x = src[i];
        put_sample(dst, d16, bf16, d32, oj + i, sdj ? __dmul_rn(scj, x) : x);
      }
    }
    if (c < C && sk == ~0u && o < dn) {  // rare: re-parse this lane's chunk from its true entry
      const StreamDesc& d = streams[s];
      const uint64_t local = (uint64_t)(c - (int64_t)d.chunk_begin);
      const uint64_t end = (local + 1) * CH;
      const uint64_t entry = local == 0 ? 0 : exit_pos[c - 1];
      Parser p;
      p.init(keys[2 * s], keys[2 * s + 1], entry);
      unsigned amb = 0;
      double x;
      uint64_t oo = o;
      double* dst = out + doff;
      uint16_t* d16 = out16 ? out16 + doff : nullptr;
      float* d32 = out32 ? out32 + doff : nullptr;
      while (p.pos < end && oo < dn) {
        if (p.attempt(z, &x, &amb)) put_sample(dst, d16, bf16, d32, oo++, scaled ? __dmul_rn(scale, x) : x);
      }
      if (amb) atomicAdd(&flags[1], amb);
    }
    __syncwarp();
  }
}

uint64_t sampler_chunks_for(uint64_t n) {
  // expected u64/sample ~1.025; + generous margin so the scan never runs short
  uint64_t pos = n + n / 8 + 4 * CH;
  return (pos + CH - 1) / CH;
}

void sampler_launch(const SamplerPlan& P, uint64_t seed, const uint64_t* d_step, uint32_t nu, double* out,
                    cudaStream_t st) {
  if (P.S == 0) return;
  k_keys<<<(P.S + 127) / 128, 128, 0, st>>>(P.d_streams, P.S, seed, d_step, nu, P.d_keys);
  unsigned grid = (unsigned)((P.C + 255) / 256);
  const bool copy = P.d_scratch && P.d_skip;
  k_spec<<<grid, 256, 0, st>>>(P.d_streams, P.d_chunk_stream, P.C, P.d_keys, P.d_spec, P.d_count,
                               copy ? P.d_scratch : nullptr, P.d_flags);
  k_scan<<<P.S, 1024, 0, st>>>(P.d_streams, P.d_keys, P.d_spec, P.d_exit, P.d_count, P.d_offset,
                               copy ? P.d_skip : nullptr, P.d_flags);
  if (copy) {
    // G chunks per warp (metadata loaded once per group): 32 for the large plans, fewer when
    // that would leave the GPU under-filled (r = 2: 23 K chunks -> 8 per warp); grid-stride,
    // up to 16 CTAs of 8 warps per SM
    int G = 32;
    while (G > 4 && (P.C + G - 1) / G < 148 * 16 * 8) G /= 2;
    const int64_t warps = (P.C + G - 1) / G;
    const unsigned cgrid = (unsigned)std::min<int64_t>((warps + 7) / 8, 148 * 16);
    k_emit_copy<<<cgrid, 256, 0, st>>>(
        P.d_streams, P.d_chunk_stream, P.C, P.d_keys, P.d_exit, P.d_offset, P.d_count, P.d_skip, P.d_scratch, out,
        static_cast<uint16_t*>(P.out16), P.out16_bf16, P.out32, G, P.d_flags);
    return;
  }
  k_emit<<<grid, 256, 0, st>>>(P.d_streams, P.d_chunk_stream, P.C, P.d_keys, P.d_exit, P.d_offset, out,
                               P.d_flags);
}

}  // namespace zo
