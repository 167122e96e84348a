// K1 sampler plan: a batch of Gaussian streams sampled in one launch sequence.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace zo {

enum StepMode : uint32_t { STEP_CURRENT = 0, STEP_WINDOW = 1, STEP_FIXED = 2 };

// One direction factor stream (StreamKey(seed, step, layer_id, role), numerics.py:139-158).
struct StreamDesc {
  uint64_t lid_hash;    // fnv1a64(utf8(layer_id))
  uint32_t role;        // Role (numerics.py:128-136)
  uint32_t step_mode;   // StepMode
  uint64_t fixed_step;  // for STEP_FIXED
  uint64_t n;           // samples (rows*cols)
  uint64_t out_off;     // element offset into the output arena
  uint64_t chunk_begin;
  uint64_t n_chunks;
  double scale;         // applied as scale*x when apply_scale (init_params: init_scale*N(0,1))
  uint32_t apply_scale;
  uint32_t seed_override;
  uint64_t seed_value;
};

struct SamplerPlan {
  int S = 0;
  int64_t C = 0;
  StreamDesc* d_streams = nullptr;
  uint32_t* d_chunk_stream = nullptr;
  uint64_t* d_keys = nullptr;
  uint64_t* d_spec = nullptr;
  uint64_t* d_exit = nullptr;
  uint32_t* d_count = nullptr;
  uint64_t* d_offset = nullptr;
  unsigned* d_flags = nullptr;  // [0] short stream, [1] exp ambiguity, [2] splice repairs
  // optional: k_spec keeps every chunk's speculative samples (C x 128 doubles) and k_scan
  // the number of leading samples to drop (d_skip; ~0u: re-parse), so the emit pass is a
  // coalesced copy instead of a second Philox + ziggurat pass
  double* d_scratch = nullptr;
  uint32_t* d_skip = nullptr;
  // optional extra outputs at the same offsets as `out`: a 16-bit (fp16 / bf16) and an fp32 copy
  void* out16 = nullptr;
  bool out16_bf16 = false;
  float* out32 = nullptr;
};

uint64_t sampler_chunks_for(uint64_t n);
void sampler_launch(const SamplerPlan& P, uint64_t seed, const uint64_t* d_step, uint32_t nu, double* out,
                    cudaStream_t st);
void host_stream_key(uint64_t seed, uint64_t step, uint64_t lid_hash, uint64_t role, uint64_t key[2]);

}  // namespace zo
