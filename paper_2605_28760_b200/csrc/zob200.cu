// libzob200 C ABI: context, device layout and the LoZO step orchestration.
//
// Device layout:
//   W64[lid]   float64 master, reference (in, out) layout -- bit-exact init/fold
//   W16T[lid]  16-bit B operand [out, in + KE] (K-major); columns in..in+3r hold
//              the window V as (hi, hi, lo) so x.W_eff = [x | t] . [W ; V]^T
//   E16        16-bit embedding [V, d] (gather + tied LM-head B operand)
//   U/V/A      float64 slot arenas in sorted layer-id order (digest order)
//   P+/P-      float32 A +- eps*U (the only sign-dependent operand)
//   activations sized for 2 * max_batch * T rows (both signs in one launch)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/zob200.h"
#include "zo_common.cuh"
#include "zo_gemm.h"
#include "zo_precise.h"
#include "zo_kernels.h"
#include "zo_sampler.h"

using namespace zo;

namespace {

thread_local std::string g_last_error;

enum Kind { K_EMBED = 0, K_QKV = 1, K_OUT = 2, K_UP = 3, K_DOWN = 4, K_POS = 5 };

struct Matrix {
  std::string lid;
  int kind = 0, layer = -1;
  int64_t m = 0, n = 0;  // reference layout: (in, out)
  uint64_t lid_hash = 0;
  int64_t u_off = 0, v_off = 0;
  int64_t z_off = 0;  // dense_mezo: offset of this matrix's z[m, n] in the dense arena
  double* W64 = nullptr;
  void* W16 = nullptr;
  int ldw = 0;
  // real32: 3xTF32 split operand [n, ldk] (projection) / [vocab, ldk] (embed), precise.cu
  float* W32S = nullptr;
  int ldk = 0;
};

struct LayerPlan {
  GemmDesc qkv, out, up, down;
  // high-rank (r > 8) tensor-core extension t = a . P_s per GEMM input and probe sign:
  // [qkv-in, out-in, up-in, down-in] x [sign]; split-K GEMMs into the fp32 workspace xws,
  // reduced in a fixed order into the activation's extension columns (ext_a / ext_ld / ext_K)
  std::vector<GemmDesc> ext;
  std::vector<void*> ext_a;
  std::vector<int> ext_ld, ext_K, ext_M, ext_neg;
  // factorized estimator: P- = -P+ exactly (A = 0), so one GEMM over both probe halves with
  // P+ and a negated finalize of the -eps rows (ext_neg = first negated row) -- 1 launch per
  // matrix instead of 2, bitwise the same t
  int ext_signs = 0;
};
// real32 (3xTF32) scorer plan: the four projections of every layer + the LM head
struct RowPlan32 {
  std::vector<GemmDesc> qkv, out, up, down;
  GemmDesc lm;
};
struct RowPlan {
  std::vector<LayerPlan> layers;
  GemmDesc lm;
  // last decoder layer past its attention, on the scored rows only (see do_score)
  bool pruned = false;
  GemmDesc last_out, last_up, last_down;
};

uint64_t fnv(const void* p, size_t n, uint64_t h) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001B3ULL;
  return h;
}
const uint64_t FNV0 = 0xCBF29CE484222325ULL;

bool env_streamk_off() {
  const char* e = std::getenv("ZO_STREAMK");
  return e && std::atoi(e) == 0;
}

struct DevAlloc {
  std::vector<void*> ptrs;
  uint64_t bytes = 0;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    size_t b = std::max<size_t>(count * sizeof(T), 256);
    ZO_CUDA_TRY(cudaMalloc(&p, b));
    ZO_CUDA_TRY(cudaMemset(p, 0, b));
    ptrs.push_back(p);
    bytes += b;
    return static_cast<T*>(p);
  }
  ~DevAlloc() {
    for (void* p : ptrs) cudaFree(p);
  }
};

}  // namespace

struct zo_ctx {
  zo_model_desc d{};
  int T = 0, Tf = 0, dh = 0, r = 0, ext_terms = 3, KE = 64, ext_used = 0, num_sms = 148;
  bool bf16 = false;
  // ZO_PREC_FP32 ("real32"): the fp32 forward on tcgen05 kind::tf32 via the 3xTF32 split
  bool real32 = false;
  // factorized dense update mode (zo_set_update_mode): false = float64 SIMT, bit-exact with the
  // reference (k_fold_dev_tiled); true = tensor-core UV^T fused into the master/shadow RMW
  // (EPI_UPDATE64, r >= 16, r % 16 == 0) -- HBM-bound, not bit-exact
  bool fast_update = false;
  // fast update mode keeps the projection / embedding masters as fp32 (in the first half of
  // each W64 allocation): 10 instead of 18 bytes per weight per update.  K_POS stays float64.
  bool master32 = false;
  float* conv_tmp = nullptr;  // CONV_CHUNK floats: in-place float64 <-> fp32 master conversion
  uint16_t *U16 = nullptr, *V16 = nullptr;  // 16-bit U / V operands of the fast update
  std::vector<GemmDesc> upd_plans;           // per matrix (empty entry: exact path)
  float *a32 = nullptr, *f32a = nullptr, *ctx32 = nullptr;  // split A operand, qkv/ff_up out, ctx
  int lda32 = 0;                                             // row stride of a32
  std::map<int, RowPlan32> plans32;
  cudaStream_t st = nullptr;
  DevAlloc mem;
  std::vector<Matrix> mats;  // sorted by lid
  int i_embed = -1;
  std::vector<int> i_qkv, i_out, i_up, i_down;
  int64_t su = 0, sv = 0;  // arena sizes
  double *U = nullptr, *V = nullptr, *A = nullptr;
  float *Pp = nullptr, *Pm = nullptr, *V32 = nullptr;
  // 1-D params (LN scale / shift) in sorted vector-id order (model.py:124-125):
  // float64 masters, full-scope directions z, and the fp32 copies the LN kernels read
  // ([0] +eps rows, [1] -eps rows; identical unless a full-scope probe is installed)
  bool full_scope = false;
  int nv = 0;
  std::vector<std::string> vids;
  std::vector<int64_t> voff, vlen;  // per 1-D param: offset / length in the vector arenas
  int64_t nvt = 0;                  // total 1-D elements
  bool opt = false;                 // ZO_ARCH_OPT
  bool dense = false;               // ZO_EST_DENSE: dense z per weight (materialising loop only)
  double* ZM = nullptr;             // dense directions of every matrix, sorted lid order
  int64_t szm = 0;
  SamplerPlan planZM;
  std::vector<StreamDesc> streamsZM;
  int i_pos = -1;                   // OPT: learned positions (offset 2)
  std::vector<float*> bqkv, bout, bup, bdown;  // OPT: fp32 bias copies per layer ([0] +eps rows)
  double *VEC64 = nullptr, *VZ = nullptr;
  float* VEC32 = nullptr;
  long vstride = 0;  // offset of the -eps copy read by the LN kernels (0: lora_only)
  SamplerPlan planZ;
  std::vector<StreamDesc> streamsZ;
  std::vector<float*> ln1g, ln1b, ln2g, ln2b;
  float *lnfg = nullptr, *lnfb = nullptr;
  // activations
  int Mmax = 0, Mpad = 0, Smax = 0, Spad = 0, ldl = 0;
  float* x32 = nullptr;
  void *hA = nullptr, *qkv = nullptr, *ctxA = nullptr, *gA = nullptr, *xs16 = nullptr;
  float *xs32 = nullptr, *z = nullptr, *logits = nullptr, *pe = nullptr;
  // scored-row copies of the last layer's activations (do_score's pruned tail)
  void *hS = nullptr, *gS = nullptr;
  float* x32S = nullptr;
  double *nll = nullptr, *out4 = nullptr, *scratch = nullptr;
  double* nll_bl = nullptr;  // materialising loop: the sign +1 NLLs while sign -1 is scored
  int64_t scratch_n = 0;
  unsigned* abort_flag = nullptr;
  int32_t *tok = nullptr, *gold = nullptr;
  uint64_t* d_step = nullptr;
  // pinned staging
  int32_t *h_tok = nullptr, *h_gold = nullptr;
  double* h_out4 = nullptr;
  uint64_t* h_step = nullptr;
  // sampler
  SamplerPlan planU, planV, planOne;
  std::vector<StreamDesc> streamsU, streamsV;
  unsigned* flags = nullptr;
  std::map<int, RowPlan> plans;  // keyed by 2*M + (nsign == 1)
  float* tpart = nullptr;         // fused LoRA-extension partials [tiles][Mpad][r]
  uint16_t* P16T = nullptr;       // high-rank extension B operands [2][su] (per matrix [r][m])
  int64_t* p16t_tab = nullptr;    // launch_p16t_all's matrix table; p16t_n entries, p16t_tiles tiles
  int p16t_n = 0, p16t_tiles = 0;
  VextMat* vext_tab = nullptr;    // write_vext_all's matrix table
  float* xws = nullptr;           // high-rank extension split-K partials [num_sms][Mpad][r]
  float* sk_ws = nullptr;         // stream-K partial tiles
  float* loss_ws = nullptr;       // k_loss per-slice partials (loss_ws_floats)
  unsigned* loss_cnt = nullptr;   // k_loss arrival counters (self-resetting)
  unsigned* sk_flags = nullptr;
  bool streamk = true;  // DP waves + stream-K tail where it pays (ZO_STREAMK=0 disables)
  int tpart_tiles = 0;
  bool fused_ext = true;
  // timing
  cudaEvent_t ev[4];
  // in-step kernel-family profile (zo_profile_step): an event before each launch group,
  // the interval up to the next mark is charged to the group's family
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev;
  std::vector<int> prof_kind;
  size_t prof_n = 0;
  float last_ms[3] = {0, 0, 0};
  double probe_eps = 0.0, probe_scale = 1.0;
  int64_t v_window = -1;  // window start whose V is loaded (-1: none)
  bool a_dirty = false;   // window A carries unfolded mass

  // captured step graph (zo_step_graph)
  cudaStream_t cap_st = nullptr;
  cudaGraphExec_t gexec = nullptr;
  struct GKey {
    uint64_t seed;
    int B, dbr;
    double eps, lr;
    bool operator==(const GKey& o) const {
      return seed == o.seed && B == o.B && dbr == o.dbr && eps == o.eps && lr == o.lr;
    }
  } gkey{};
  bool gkey_valid = false;
  int graph_kernels = 0;  // kernel nodes of the captured step body
  // captured halves of the multi-GPU step (zo_step_score_graph / zo_step_apply_graph,
  // zo_qdir_*_graph): the collective runs between two graph launches
  struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    std::vector<uint64_t> key;
    bool valid = false;
    int kernels = 0;
  };
  GraphSlot gs_score, gs_apply, gs_qscore, gs_qapply;
  // asynchronous slot snapshots (zo_slot_snapshot): U / V -> a device copy (in stream order)
  // -> pinned host ring on a side stream, overlapping the next step
  static constexpr int SNAP_RING = 4;
  cudaStream_t snap_st = nullptr;
  double* snap_dev[2] = {nullptr, nullptr};
  double* snap_host[2][SNAP_RING] = {};
  bool snap_taken[2][SNAP_RING] = {};  // a snapshot was started into the slot
  cudaEvent_t snap_ready[2][SNAP_RING] = {}, snap_done[2][SNAP_RING] = {};
  cudaEvent_t snap_last[2] = {nullptr, nullptr};  // the last D2H out of snap_dev[which]
  uint64_t* d_base = nullptr;  // q-direction macro-step base step (t * G), set before the apply graph
  void drop_graphs() {
    gkey_valid = false;
    for (GraphSlot* g : {&gs_score, &gs_apply, &gs_qscore, &gs_qapply}) g->valid = false;
  }

  ~zo_ctx() {
    if (gexec) cudaGraphExecDestroy(gexec);
    for (GraphSlot* g : {&gs_score, &gs_apply, &gs_qscore, &gs_qapply})
      if (g->exec) cudaGraphExecDestroy(g->exec);
    for (int w = 0; w < 2; ++w)
      for (int k = 0; k < SNAP_RING; ++k) {
        if (snap_host[w][k]) cudaFreeHost(snap_host[w][k]);
        if (snap_ready[w][k]) cudaEventDestroy(snap_ready[w][k]);
        if (snap_done[w][k]) cudaEventDestroy(snap_done[w][k]);
      }
    if (snap_st) cudaStreamDestroy(snap_st);
    if (cap_st) cudaStreamDestroy(cap_st);
    if (h_tok) cudaFreeHost(h_tok);
    if (h_gold) cudaFreeHost(h_gold);
    if (h_out4) cudaFreeHost(h_out4);
    if (h_step) cudaFreeHost(h_step);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : prof_ev) cudaEventDestroy(e);
  }
};

namespace zo {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ZO_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
}  // namespace zo

namespace {

__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }
__global__ void k_step_from_base(uint64_t* step, const uint64_t* base, uint64_t g) { *step = *base + g; }

int fail(const Error& e) {
  g_last_error = e.msg;
  return e.code;
}

#define ZO_API_BEGIN try {
#define ZO_API_END                                                   \
  }                                                                  \
  catch (const Error& e) { return fail(e); }                         \
  catch (const std::exception& e) { return fail(Error(ZO_ERR_INTERNAL, e.what())); }

void check(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

Matrix& find(zo_ctx* c, const char* lid) {
  for (auto& m : c->mats)
    if (m.lid == lid) return m;
  throw Error(ZO_ERR_INPUT, std::string("unknown layer id ") + lid);
}

void build_sampler_plan(zo_ctx* c, SamplerPlan& P, std::vector<StreamDesc>& sd, bool scratch = false) {
  int64_t chunk = 0;
  std::vector<uint32_t> chunk_stream;
  for (size_t s = 0; s < sd.size(); ++s) {
    sd[s].chunk_begin = (uint64_t)chunk;
    sd[s].n_chunks = sampler_chunks_for(sd[s].n);
    for (uint64_t i = 0; i < sd[s].n_chunks; ++i) chunk_stream.push_back((uint32_t)s);
    chunk += (int64_t)sd[s].n_chunks;
  }
  P.S = (int)sd.size();
  P.C = chunk;
  P.d_streams = c->mem.get<StreamDesc>(sd.size());
  P.d_chunk_stream = c->mem.get<uint32_t>(chunk);
  P.d_keys = c->mem.get<uint64_t>(2 * sd.size());
  P.d_spec = c->mem.get<uint64_t>(chunk);
  P.d_exit = c->mem.get<uint64_t>(chunk);
  P.d_count = c->mem.get<uint32_t>(chunk);
  P.d_offset = c->mem.get<uint64_t>(chunk);
  P.d_flags = c->flags;
  if (scratch) {  // speculative samples kept for the copy emit (zo_sampler.h)
    P.d_scratch = c->mem.get<double>((size_t)chunk * 128);
    P.d_skip = c->mem.get<uint32_t>(chunk);
  }
  ZO_CUDA_TRY(cudaMemcpy(P.d_streams, sd.data(), sd.size() * sizeof(StreamDesc), cudaMemcpyHostToDevice));
  ZO_CUDA_TRY(cudaMemcpy(P.d_chunk_stream, chunk_stream.data(), chunk_stream.size() * 4, cudaMemcpyHostToDevice));
}

// OPT biases in a GEMM epilogue; rows of the -eps probe read the second fp32 copy
// (the VectorProbe -1 values under full scope, identical otherwise)
void set_bias(const zo_ctx* c, GemmDesc& g, const float* bias, int rows_per_sign) {
  g.bias = bias;
  g.bias_rps = rows_per_sign;
  g.bias_vstride = c->vstride;
}

// high-rank extension of a factorized probe pair: one GEMM for both signs (LayerPlan::ext_signs)
bool ext_merged(const zo_ctx* c, int nsign) {
  return !c->fused_ext && nsign == 2 && c->d.estimator == ZO_EST_FACTORIZED && !c->full_scope;
}

RowPlan& row_plan(zo_ctx* c, int M, int nsign = 2) {
  const int key = 2 * M + (nsign == 1 ? 1 : 0);
  auto it = c->plans.find(key);
  if (it != c->plans.end()) return it->second;
  RowPlan rp;
  const int d = c->d.dim;
  const int ldh = d + c->KE, ldg = 4 * d + c->KE;
  const int S = M / c->Tf * c->d.opt_len;
  for (int l = 0; l < c->d.n_layers; ++l) {
    LayerPlan lp;
    const Matrix& q = c->mats[c->i_qkv[l]];
    const Matrix& o = c->mats[c->i_out[l]];
    const Matrix& u = c->mats[c->i_up[l]];
    const Matrix& w = c->mats[c->i_down[l]];
    gemm_plan(lp.qkv, c->hA, M, ldh, q.W16, 3 * d, q.ldw, d + c->ext_used, EPI_STORE16, c->bf16, c->qkv, 3 * d,
              c->num_sms);
    gemm_plan(lp.out, c->ctxA, M, ldh, o.W16, d, o.ldw, d + c->ext_used, EPI_RESID32, c->bf16, c->x32, d,
              c->num_sms);
    gemm_plan(lp.up, c->hA, M, ldh, u.W16, 4 * d, u.ldw, d + c->ext_used,
              c->fused_ext ? EPI_GELU16_EXT : EPI_GELU16, c->bf16, c->gA, ldg, c->num_sms);
    if (c->fused_ext) {
      lp.up.xPp = c->Pp + w.u_off;
      lp.up.xPm = c->Pm + w.u_off;
      lp.up.xr = c->r;
      lp.up.xrps = M / nsign;
      lp.up.tpart_ld = c->Mpad;
      lp.up.tpart = c->tpart;
      check(gemm_ext_slots(lp.up, 4 * d) <= c->tpart_tiles, ZO_ERR_INTERNAL, "tpart too small");
    }
    gemm_plan(lp.down, c->gA, M, ldg, w.W16, d, w.ldw, 4 * d + c->ext_used, EPI_RESID32, c->bf16, c->x32, d,
              c->num_sms);
    set_bias(c, lp.qkv, c->bqkv[l], M / nsign);
    set_bias(c, lp.out, c->bout[l], M / nsign);
    set_bias(c, lp.up, c->bup[l], M / nsign);
    set_bias(c, lp.down, c->bdown[l], M / nsign);
    lp.up.relu = c->opt ? 1 : 0;
    if (c->streamk)
      for (GemmDesc* g : {&lp.qkv, &lp.out, &lp.up, &lp.down}) gemm_enable_streamk(*g, c->sk_ws, c->sk_flags, c->num_sms);
    for (GemmDesc* g : {&lp.qkv, &lp.out, &lp.up, &lp.down}) gemm_enable_halftail(*g, c->num_sms);
    if (!c->fused_ext) {
      const int rps = M / nsign;
      const Matrix* mm[4] = {&q, &o, &u, &w};
      void* acts[4] = {c->hA, c->ctxA, c->hA, c->gA};
      const int lds[4] = {ldh, ldh, ldh, ldg};
      lp.ext.resize(8);
      lp.ext_a.resize(8);
      lp.ext_ld.resize(8);
      lp.ext_K.resize(8);
      lp.ext_M.resize(8);
      lp.ext_neg.resize(8);
      const bool merged = ext_merged(c, nsign);
      lp.ext_signs = merged ? 1 : nsign;
      const int mext = merged ? 2 * rps : rps;
      for (int i = 0; i < 4; ++i)
        for (int sg = 0; sg < lp.ext_signs; ++sg) {
          uint16_t* a = static_cast<uint16_t*>(acts[i]) + (size_t)sg * rps * lds[i];
          GemmDesc& g = lp.ext[2 * i + sg];
          // t = a . P_s: a few output tiles over K = 5120 .. 20480 -- split K so every SM works
          // one N tile per rank block (r <= 128: A read once, the split-K partials fill the SMs)
          gemm_plan(g, a, mext, lds[i], c->P16T + (size_t)sg * c->su + mm[i]->u_off, c->r, (int)mm[i]->m,
                    (int)mm[i]->m, EPI_STORE32, c->bf16, c->xws, c->r, c->num_sms, c->r <= 128 ? 128 : 0);
          const int tiles = ((mext + 127) / 128) * ((c->r + g.bn - 1) / g.bn);
          gemm_enable_splitk(g, std::max(1, c->num_sms / tiles), (long)c->Mpad * c->r);
          lp.ext_a[2 * i + sg] = a;
          lp.ext_ld[2 * i + sg] = lds[i];
          lp.ext_K[2 * i + sg] = (int)mm[i]->m;
          lp.ext_M[2 * i + sg] = mext;
          lp.ext_neg[2 * i + sg] = merged ? rps : -1;
        }
    }
    rp.layers.push_back(lp);
  }
  const Matrix& e = c->mats[c->i_embed];
  gemm_plan(rp.lm, c->xs16, S, d, e.W16, c->d.vocab, d, d, EPI_STORE32, c->bf16, c->logits, c->ldl, c->num_sms);
  // Only the scored rows (prompt_len-1+j) reach the loss, and causal attention makes
  // every other row's last-layer output irrelevant: past the last attention, run
  // attn_out / LN2 / FFN on those S rows (weight-read-bound small-M GEMMs) instead of
  // all M.  The fused-extension path (r <= 8) only.
  if (c->fused_ext && c->d.n_layers > 0) {
    const int L = c->d.n_layers - 1;
    const Matrix& o = c->mats[c->i_out[L]];
    const Matrix& u = c->mats[c->i_up[L]];
    const Matrix& w = c->mats[c->i_down[L]];
    gemm_plan(rp.last_out, c->hS, S, ldh, o.W16, d, o.ldw, d + c->ext_used, EPI_RESID32, c->bf16, c->x32S, d,
              c->num_sms);
    gemm_plan(rp.last_up, c->hS, S, ldh, u.W16, 4 * d, u.ldw, d + c->ext_used, EPI_GELU16_EXT, c->bf16, c->gS, ldg,
              c->num_sms);
    rp.last_up.xPp = c->Pp + w.u_off;
    rp.last_up.xPm = c->Pm + w.u_off;
    rp.last_up.xr = c->r;
    rp.last_up.xrps = S / nsign;
    rp.last_up.tpart_ld = c->Mpad;
    rp.last_up.tpart = c->tpart;
    gemm_plan(rp.last_down, c->gS, S, ldg, w.W16, d, w.ldw, 4 * d + c->ext_used, EPI_RESID32, c->bf16, c->x32S, d,
              c->num_sms);
    set_bias(c, rp.last_out, c->bout[L], S / nsign);
    set_bias(c, rp.last_up, c->bup[L], S / nsign);
    set_bias(c, rp.last_down, c->bdown[L], S / nsign);
    rp.last_up.relu = c->opt ? 1 : 0;
    rp.pruned = true;
  }
  return c->plans.emplace(key, std::move(rp)).first->second;
}

void refresh_shadow(zo_ctx* c, const Matrix& m) {
  if (m.kind == K_POS) return;
  if (m.kind == K_EMBED)
    launch_shadow(m.W64, m.m * m.n, m.W16, c->bf16, c->st);
  else
    launch_shadow_T(m.W64, (int)m.m, (int)m.n, m.W16, m.ldw, c->bf16, c->st);
}

// In-place master conversion, chunk by chunk through conv_tmp (stream-ordered): narrowing
// walks up (chunk k's fp32 bytes [4kC, 4kC+4C) only overwrite float64 chunks < k, already
// read), widening walks down (chunk k's float64 bytes only overwrite fp32 chunks >= k).
constexpr int64_t CONV_CHUNK = 1 << 24;
bool has_master32(const Matrix& m) { return m.kind != K_POS; }
void narrow_master(zo_ctx* c, Matrix& m) {
  const int64_t n = m.m * m.n;
  float* dst = reinterpret_cast<float*>(m.W64);
  for (int64_t o = 0; o < n; o += CONV_CHUNK) {
    const int64_t k = std::min(CONV_CHUNK, n - o);
    launch_f64_to_f32(m.W64 + o, c->conv_tmp, k, c->st);
    ZO_CUDA_TRY(cudaMemcpyAsync(dst + o, c->conv_tmp, (size_t)k * 4, cudaMemcpyDeviceToDevice, c->st));
  }
}
void widen_master(zo_ctx* c, Matrix& m) {
  const int64_t n = m.m * m.n;
  const float* src = reinterpret_cast<const float*>(m.W64);
  for (int64_t o = ((n - 1) / CONV_CHUNK) * CONV_CHUNK; o >= 0; o -= CONV_CHUNK) {
    const int64_t k = std::min(CONV_CHUNK, n - o);
    ZO_CUDA_TRY(cudaMemcpyAsync(c->conv_tmp, src + o, (size_t)k * 4, cudaMemcpyDeviceToDevice, c->st));
    launch_f32_to_f64(c->conv_tmp, m.W64 + o, k, c->st);
  }
}
// run f on a float64 view of m's master (widen -> f -> narrow when the master is fp32)
template <class F>
void with_master64(zo_ctx* c, Matrix& m, F&& f) {
  const bool conv = c->master32 && has_master32(m);
  if (conv) widen_master(c, m);
  f();
  if (conv) narrow_master(c, m);
}

void write_vext_all(zo_ctx* c) {
  if (!c->vext_tab) {  // one table for the batched launch (matrix order = V arena order)
    std::vector<VextMat> tab;
    for (auto& m : c->mats) tab.push_back({m.v_off, m.kind == K_EMBED ? nullptr : m.W16, m.ldw, (int)m.m});
    c->vext_tab = c->mem.get<VextMat>(tab.size());
    ZO_CUDA_TRY(cudaMemcpy(c->vext_tab, tab.data(), tab.size() * sizeof(VextMat), cudaMemcpyHostToDevice));
  }
  launch_write_vext_all(c->V, c->sv, c->vext_tab, (int)c->mats.size(), c->r, c->bf16, c->ext_terms, c->V32, c->st);
}

enum ProfKind { PK_EMBED = 0, PK_LN, PK_QKV, PK_ATTN, PK_EXT, PK_OUT, PK_UP, PK_DOWN, PK_TAIL, PK_OTHER, PK_N };
void prof_mark(zo_ctx* c, int kind) {
  if (!c->prof_on) return;
  if (c->prof_n == c->prof_ev.size()) {
    cudaEvent_t e;
    ZO_CUDA_TRY(cudaEventCreate(&e));
    c->prof_ev.push_back(e);
    c->prof_kind.push_back(0);
  }
  ZO_CUDA_TRY(cudaEventRecord(c->prof_ev[c->prof_n], c->st));
  c->prof_kind[c->prof_n++] = kind;
}

RowPlan32& row_plan32(zo_ctx* c, int M, int nsign) {
  const int key = 2 * M + (nsign == 1 ? 1 : 0);
  auto it = c->plans32.find(key);
  if (it != c->plans32.end()) return it->second;
  RowPlan32 rp;
  const int d = c->d.dim, r = c->r, S = M / c->Tf * c->d.opt_len;
  const int ld_d = (int)ceil_div(3 * d + 3 * r, 32) * 32, ld_4d = (int)ceil_div(12 * d + 3 * r, 32) * 32;
  for (int l = 0; l < c->d.n_layers; ++l) {
    const Matrix& q = c->mats[c->i_qkv[l]];
    const Matrix& o = c->mats[c->i_out[l]];
    const Matrix& u = c->mats[c->i_up[l]];
    const Matrix& w = c->mats[c->i_down[l]];
    GemmDesc gq, go, gu, gd;
    gemm_plan(gq, c->a32, M, ld_d, q.W32S, 3 * d, q.ldk, 3 * d + 3 * r, EPI_STORE32, 2, c->f32a, 3 * d, c->num_sms);
    gemm_plan(go, c->a32, M, ld_d, o.W32S, d, o.ldk, 3 * d + 3 * r, EPI_RESID32, 2, c->x32, d, c->num_sms);
    gemm_plan(gu, c->a32, M, ld_d, u.W32S, 4 * d, u.ldk, 3 * d + 3 * r, EPI_STORE32, 2, c->f32a, 4 * d,
              c->num_sms);
    gemm_plan(gd, c->a32, M, ld_4d, w.W32S, d, w.ldk, 12 * d + 3 * r, EPI_RESID32, 2, c->x32, d, c->num_sms);
    set_bias(c, gq, c->bqkv[l], M / nsign);
    set_bias(c, go, c->bout[l], M / nsign);
    set_bias(c, gu, c->bup[l], M / nsign);
    set_bias(c, gd, c->bdown[l], M / nsign);
    rp.qkv.push_back(gq);
    rp.out.push_back(go);
    rp.up.push_back(gu);
    rp.down.push_back(gd);
  }
  const Matrix& e = c->mats[c->i_embed];
  gemm_plan(rp.lm, c->a32, S, e.ldk, e.W32S, c->d.vocab, e.ldk, 3 * d, EPI_STORE32, 2, c->logits, c->ldl,
            c->num_sms);
  return c->plans32.emplace(key, std::move(rp)).first->second;
}

// the reference's "real32" forward (model.py:149-199, float32 arithmetic) on the tensor cores:
// 3xTF32 split GEMMs with the LoRA term as extension K columns, fp32 LN / attention / GELU
// (precise.cu); the embedding, final LN and loss kernels are the 16-bit path's fp32 ones.
void do_score32(zo_ctx* c, int B, int nsign) {
  const int d = c->d.dim, T = c->Tf, M = nsign * B * T, r = c->r, rps = B * T;
  // split operands from the float64 masters and the current window V (every call: folds,
  // dense updates and uploads all land in W64 / V)
  for (const auto& m : c->mats)
    if (m.W32S)
      launch_split_weight(m.W64, (int)m.m, (int)m.n, c->V + m.v_off, r, m.W32S, m.ldk, m.kind == K_EMBED ? 0 : 1,
                          c->st);
  RowPlan32& rp = row_plan32(c, M, nsign);
  const Matrix& e = c->mats[c->i_embed];
  const int ld_d = (int)ceil_div(3 * d + 3 * r, 32) * 32, ld_4d = (int)ceil_div(12 * d + 3 * r, 32) * 32;
  PosEmbed pos;
  if (c->opt) {
    const Matrix& pm = c->mats[c->i_pos];
    pos.W64 = pm.W64;
    pos.Pp = c->Pp + pm.u_off;
    pos.Pm = c->Pm + pm.u_off;
    pos.V32 = c->V32 + pm.v_off;
    pos.offset = 2;
  }
  launch_embed(c->x32, c->tok, c->T, B, T, d, e.W64, nullptr, e.W16, false, c->Pp + e.u_off, c->Pm + e.u_off,
               c->V32 + e.v_off, r, c->pe, pos, M, c->st);
  for (int l = 0; l < c->d.n_layers; ++l) {
    const Matrix& q = c->mats[c->i_qkv[l]];
    const Matrix& o = c->mats[c->i_out[l]];
    const Matrix& u = c->mats[c->i_up[l]];
    const Matrix& w = c->mats[c->i_down[l]];
    launch_ln_split(c->x32, c->ln1g[l], c->ln1b[l], c->vstride, M, d, c->a32, ld_d, c->Pp + q.u_off,
                    c->Pm + q.u_off, r, rps, c->st);
    gemm_launch(rp.qkv[l], c->st);
    launch_attn32(c->f32a, 3 * d, c->ctx32, d, nsign * B, T, c->d.n_heads, c->dh, c->st);
    launch_split_act(c->ctx32, d, M, d, c->a32, ld_d, c->Pp + o.u_off, c->Pm + o.u_off, r, rps, 0, c->st);
    gemm_launch(rp.out[l], c->st);
    launch_ln_split(c->x32, c->ln2g[l], c->ln2b[l], c->vstride, M, d, c->a32, ld_d, c->Pp + u.u_off,
                    c->Pm + u.u_off, r, rps, c->st);
    gemm_launch(rp.up[l], c->st);
    launch_split_act(c->f32a, 4 * d, M, 4 * d, c->a32, ld_4d, c->Pp + w.u_off, c->Pm + w.u_off, r, rps,
                     c->opt ? 2 : 1, c->st);
    gemm_launch(rp.down[l], c->st);
  }
  const int S = nsign * B * c->d.opt_len;
  launch_final_ln(c->x32, c->lnfg, c->lnfb, B * nsign, T, d, c->d.prompt_len, c->d.opt_len, c->xs32, c->xs16,
                  false, c->V32 + e.v_off, r, c->z, rps, c->vstride, c->st);
  launch_split_act(c->xs32, d, S, d, c->a32, e.ldk, nullptr, nullptr, 0, S, 0, c->st);
  gemm_launch(rp.lm, c->st);
  launch_loss(c->logits, c->ldl, c->d.vocab, c->z, r, c->Pp + e.u_off, c->Pm + e.u_off, c->gold, B,
              c->d.opt_len, c->loss_ws, c->loss_cnt, c->nll, c->st);
}

void do_score(zo_ctx* c, int B, int nsign) {
  const int d = c->d.dim, T = c->Tf, M = nsign * B * T;
  check(B >= 1 && B <= c->d.max_batch, ZO_ERR_DIMENSION, "batch size out of range");
  if (c->real32) {
    do_score32(c, B, nsign);
    return;
  }
  RowPlan& rp = row_plan(c, M, nsign);
  const Matrix& e = c->mats[c->i_embed];
  const int rps = B * T;
  const int ldh = d + c->KE, ldg = 4 * d + c->KE;
  PosEmbed pos;
  if (c->opt) {  // learned positions at offset 2 (+ their LoRA delta)
    const Matrix& pm = c->mats[c->i_pos];
    pos.W64 = pm.W64;
    pos.Pp = c->Pp + pm.u_off;
    pos.Pm = c->Pm + pm.u_off;
    pos.V32 = c->V32 + pm.v_off;
    pos.offset = 2;
  }
  prof_mark(c, PK_EMBED);
  launch_embed(c->x32, c->tok, c->T, B, T, d, c->master32 ? nullptr : e.W64,
               c->master32 ? reinterpret_cast<const float*>(e.W64) : nullptr, e.W16, c->bf16, c->Pp + e.u_off,
               c->Pm + e.u_off, c->V32 + e.v_off,
               c->r, c->pe, pos, M, c->st);
  if (!c->fused_ext)  // high rank: 16-bit transposed probe operands of the extension GEMMs
    launch_p16t_all(c->Pp, c->Pm, c->su, c->p16t_tab, c->p16t_n, c->p16t_tiles, c->r, ext_merged(c, nsign) ? 1 : nsign,
                    c->P16T, c->bf16, c->st);
  auto ext_gemm = [&](const LayerPlan& lp, int i) {
    for (int sg = 0; sg < lp.ext_signs; ++sg) {
      const int j = 2 * i + sg;
      gemm_launch(lp.ext[j], c->st);
      launch_ext_finalize(c->xws, lp.ext[j].ksplit, c->Mpad, lp.ext_M[j], c->r, lp.ext_a[j], lp.ext_ld[j],
                          lp.ext_K[j], 1, c->bf16, c->st, lp.ext_neg[j]);
    }
  };
  for (int l = 0; l < c->d.n_layers; ++l) {
    const Matrix& q = c->mats[c->i_qkv[l]];
    const Matrix& o = c->mats[c->i_out[l]];
    const Matrix& u = c->mats[c->i_up[l]];
    const Matrix& w = c->mats[c->i_down[l]];
    const LayerPlan& lp = rp.layers[l];
    prof_mark(c, PK_LN);
    launch_ln_ext(c->x32, c->ln1g[l], c->ln1b[l], M, d, c->hA, ldh, c->bf16, c->Pp + q.u_off, c->Pm + q.u_off,
                  c->fused_ext ? c->r : 0, rps, c->ext_terms, c->vstride, c->st);
    if (!c->fused_ext) ext_gemm(lp, 0);
    prof_mark(c, PK_QKV);
    gemm_launch(lp.qkv, c->st);
    AttnExt ax;
    if (c->fused_ext) {
      ax.Pp = c->Pp + o.u_off;
      ax.Pm = c->Pm + o.u_off;
      ax.r = c->r;
      ax.rps = rps;
      ax.ld = c->Mpad;
      ax.tpart = c->tpart;
    }
    prof_mark(c, PK_ATTN);
    launch_attention(c->qkv, 3 * d, c->ctxA, ldh, nsign * B, T, c->d.n_heads, c->dh, c->bf16, ax, c->st);
    if (rp.pruned && l == c->d.n_layers - 1) {
      // scored rows only from here (RowPlan::pruned): compact ctx (+ extension columns)
      // and residual rows, then attn_out / LN2 / FFN on S rows
      const int S = nsign * B * c->d.opt_len;
      prof_mark(c, PK_TAIL);
      launch_ext_finalize(c->tpart, c->d.n_heads, c->Mpad, M, c->r, c->ctxA, ldh, d, c->ext_terms, c->bf16, c->st);
      launch_gather_scored(c->ctxA, (size_t)ldh * 2, c->hS, (size_t)ldh * 2, ldh * 2, nsign, B, T, c->d.prompt_len,
                           c->d.opt_len, c->st);
      launch_gather_scored(c->x32, (size_t)d * 4, c->x32S, (size_t)d * 4, d * 4, nsign, B, T, c->d.prompt_len,
                           c->d.opt_len, c->st);
      gemm_launch(rp.last_out, c->st);
      launch_ln_ext(c->x32S, c->ln2g[l], c->ln2b[l], S, d, c->hS, ldh, c->bf16, c->Pp + u.u_off, c->Pm + u.u_off,
                    c->r, S / nsign, c->ext_terms, c->vstride, c->st);
      gemm_launch(rp.last_up, c->st);
      launch_ext_finalize(c->tpart, gemm_ext_slots(rp.last_up, 4 * d), c->Mpad, S, c->r, c->gS, ldg,
                          4 * d, c->ext_terms, c->bf16, c->st);
      gemm_launch(rp.last_down, c->st);
      break;
    }
    prof_mark(c, PK_EXT);
    if (c->fused_ext)
      launch_ext_finalize(c->tpart, c->d.n_heads, c->Mpad, M, c->r, c->ctxA, ldh, d, c->ext_terms, c->bf16, c->st);
    else
      ext_gemm(lp, 1);
    prof_mark(c, PK_OUT);
    gemm_launch(lp.out, c->st);
    prof_mark(c, PK_LN);
    launch_ln_ext(c->x32, c->ln2g[l], c->ln2b[l], M, d, c->hA, ldh, c->bf16, c->Pp + u.u_off, c->Pm + u.u_off,
                  c->fused_ext ? c->r : 0, rps, c->ext_terms, c->vstride, c->st);
    if (!c->fused_ext) ext_gemm(lp, 2);
    prof_mark(c, PK_UP);
    gemm_launch(lp.up, c->st);
    prof_mark(c, PK_EXT);
    if (c->fused_ext)
      launch_ext_finalize(c->tpart, gemm_ext_slots(lp.up, 4 * d), c->Mpad, M, c->r, c->gA, ldg, 4 * d,
                          c->ext_terms, c->bf16, c->st);
    else
      ext_gemm(lp, 3);
    prof_mark(c, PK_DOWN);
    gemm_launch(lp.down, c->st);
  }
  prof_mark(c, PK_TAIL);
  if (rp.pruned)  // x32S rows are already the scored rows, in [sign][b][j] order
    launch_final_ln(c->x32S, c->lnfg, c->lnfb, B * nsign, c->d.opt_len, d, 1, c->d.opt_len, c->xs32, c->xs16,
                    c->bf16, c->V32 + e.v_off, c->r, c->z, B * c->d.opt_len, c->vstride, c->st);
  else
    launch_final_ln(c->x32, c->lnfg, c->lnfb, B * nsign, T, d, c->d.prompt_len, c->d.opt_len, c->xs32, c->xs16,
                    c->bf16, c->V32 + e.v_off, c->r, c->z, rps, c->vstride, c->st);
  gemm_launch(rp.lm, c->st);
  launch_loss(c->logits, c->ldl, c->d.vocab, c->z, c->r, c->Pp + e.u_off, c->Pm + e.u_off, c->gold, B,
              c->d.opt_len, c->loss_ws, c->loss_cnt, c->nll, c->st);
}

// gold: [gold_signs, B, opt_len]; with gold_signs == 1 both probe halves share it
void stage_batch(zo_ctx* c, const int32_t* tokens, const int32_t* gold, int B, int gold_signs) {
  const size_t nt = (size_t)B * c->T, ng = (size_t)gold_signs * B * c->d.opt_len;
  for (size_t i = 0; i < nt; ++i)
    check(tokens[i] >= 0 && tokens[i] < c->d.vocab, ZO_ERR_INPUT,
          "token id outside [0, " + std::to_string(c->d.vocab) + ")");
  for (size_t i = 0; i < ng; ++i)
    check(gold[i] >= 0 && gold[i] < c->d.vocab, ZO_ERR_INPUT, "gold token id out of range");
  std::memcpy(c->h_tok, tokens, nt * 4);
  std::memcpy(c->h_gold, gold, ng * 4);
  if (gold_signs == 1) std::memcpy(c->h_gold + ng, gold, ng * 4);
  ZO_CUDA_TRY(cudaMemcpyAsync(c->tok, c->h_tok, nt * 4, cudaMemcpyHostToDevice, c->st));
  ZO_CUDA_TRY(cudaMemcpyAsync(c->gold, c->h_gold, 2 * (ng / gold_signs) * 4, cudaMemcpyHostToDevice, c->st));
}

void set_step(zo_ctx* c, uint64_t step) {
  // pinned staging is reused: wait for the previous copy to drain before overwriting
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  *c->h_step = step;
  ZO_CUDA_TRY(cudaMemcpyAsync(c->d_step, c->h_step, 8, cudaMemcpyHostToDevice, c->st));
}

void launch_dense_update_dev(zo_ctx* c, double lr, const double* out4, const unsigned* abort_flag) {
  if (c->fast_update) {
    // 16-bit operands of this step's directions (written by the sampler's emit when its plans
    // carry them, else converted here), then one fused GEMM + RMW per matrix
    if (c->planU.out16 != c->U16) launch_shadow(c->U, c->su, c->U16, c->bf16, c->st);
    if (c->planV.out16 != c->V16) launch_shadow(c->V, c->sv, c->V16, c->bf16, c->st);
    if (c->upd_plans.empty()) {
      c->upd_plans.resize(c->mats.size());
      for (size_t i = 0; i < c->mats.size(); ++i) {
        const Matrix& m = c->mats[i];
        if (m.kind == K_POS) continue;  // no 16-bit shadow: the exact path below
        GemmDesc& g = c->upd_plans[i];
        // D = V U^T (rows = outputs j): the master W[i][j] is then read / written with the lanes
        // along j (coalesced) -- projections, and the embedding too when its master is fp32
        // (its shadow E16[i][j] is row-major: upd_shadow_rm)
        const bool tr = m.kind != K_EMBED || c->master32;
        if (tr)  // D[j, i] = sum_k V[j, k] U[i, k]: rows = outputs (W16T rows)
          gemm_plan(g, c->V16 + m.v_off, (int)m.n, c->r, c->U16 + m.u_off, (int)m.m, c->r, c->r, EPI_UPDATE64,
                    c->bf16, nullptr, 0, c->num_sms);
        else
          gemm_plan(g, c->U16 + m.u_off, (int)m.m, c->r, c->V16 + m.v_off, (int)m.n, c->r, c->r, EPI_UPDATE64,
                    c->bf16, nullptr, 0, c->num_sms);
        g.upd_w64 = m.W64;
        g.upd_m32 = c->master32 ? 1 : 0;
        g.upd_w16 = m.W16;
        g.upd_ld64 = (int)m.n;
        g.upd_ld16 = m.kind == K_EMBED ? (int)m.n : m.ldw;
        g.upd_transposed = tr ? 1 : 0;
        g.upd_shadow_rm = (tr && m.kind == K_EMBED) ? 1 : 0;
        g.upd_lr = lr;
        g.upd_scale = 1.0 / std::sqrt((double)c->r);
        gemm_set_update_master(g);
      }
    }
    for (size_t i = 0; i < c->mats.size(); ++i) {
      const Matrix& m = c->mats[i];
      if (m.kind == K_POS) {
        launch_fold_dev(m.W64, (int)m.m, (int)m.n, c->U + m.u_off, c->V + m.v_off, c->r, out4, lr,
                        1.0 / std::sqrt((double)c->r), abort_flag, m.W16, (int)m.n, 0, c->bf16, c->st);
        continue;
      }
      c->upd_plans[i].upd_lr = lr;
      c->upd_plans[i].upd_out4 = out4;
      c->upd_plans[i].upd_abort = abort_flag;
      gemm_launch(c->upd_plans[i], c->st);
    }
    return;
  }
  for (auto& m : c->mats)
    launch_fold_dev(m.W64, (int)m.m, (int)m.n, c->U + m.u_off, c->V + m.v_off, c->r, out4, lr,
                    1.0 / std::sqrt((double)c->r), abort_flag, m.W16, m.kind == K_EMBED ? (int)m.n : m.ldw,
                    m.kind == K_EMBED ? 0 : 1, c->bf16, c->st);
}

// full scope: fp32 LN copies for the probe pair (eps) or the plain params (eps = 0)
void vec_probe(zo_ctx* c, double eps) {
  if (c->full_scope) launch_vec_probe(c->VEC64, c->VZ, c->nvt, eps, c->VEC32, c->st);
}
// full scope: VectorProbe.update with the coefficient in out4 (device)
void vec_update(zo_ctx* c, const double* out4, double lr, const unsigned* abort_flag) {
  if (c->full_scope)
    launch_vec_update(c->VEC64, c->VZ, c->nvt, out4, lr, abort_flag, c->VEC32, c->st);
}
void sample_z(zo_ctx* c, uint64_t seed) {
  if (c->full_scope) sampler_launch(c->planZ, seed, c->d_step, 1, c->VZ, c->st);
}

void fold_all(zo_ctx* c) {
  for (auto& m : c->mats)
    launch_fold(m.W64, (int)m.m, (int)m.n, c->A + m.u_off, c->V + m.v_off, c->r, 1.0, m.W16,
                m.kind == K_EMBED ? (int)m.n : m.ldw, m.kind == K_EMBED ? 0 : 1, c->bf16, c->st);
  ZO_CUDA_TRY(cudaMemsetAsync(c->A, 0, (size_t)c->su * 8, c->st));
  c->a_dirty = false;
}

}  // namespace

static void graph_body(zo_ctx* c, uint64_t seed, double eps, double lr, int32_t divide_by_r, int32_t B);

extern "C" {

const char* zo_last_error(void) { return g_last_error.c_str(); }
int zo_version(void) { return 1; }

int zo_create(zo_ctx** out, const zo_model_desc* desc) {
  ZO_API_BEGIN
  check(out && desc, ZO_ERR_CONFIG, "null argument");
  const zo_model_desc& d = *desc;
  check(d.dim % d.n_heads == 0, ZO_ERR_CONFIG, "dim not divisible by n_heads");
  check(d.vocab >= 8, ZO_ERR_CONFIG, "vocab must be >= 8");
  check(d.dim % 8 == 0, ZO_ERR_DIMENSION, "dim must be a multiple of 8 for the tensor-core path");
  check(d.rank >= 1 && d.max_batch >= 1 && d.opt_len >= 1 && d.prompt_len >= 1, ZO_ERR_CONFIG, "bad sizes");
  check(d.prompt_len + d.opt_len <= 128, ZO_ERR_DIMENSION, "sequence length > 128 not supported");
  std::unique_ptr<zo_ctx> c(new zo_ctx());
  c->d = d;
  ZO_CUDA_TRY(cudaSetDevice(d.device));
  cudaDeviceProp prop;
  ZO_CUDA_TRY(cudaGetDeviceProperties(&prop, d.device));
  check(prop.major == 10, ZO_ERR_CUDA, std::string("libzob200 targets sm_100a (B200); found ") + prop.name);
  c->num_sms = prop.multiProcessorCount;
  c->T = d.prompt_len + d.opt_len;
  // the forward runs positions [0, T-1): the last token is never attended by a scored row
  // (rows prompt_len-1+j, j < opt_len, are causal), so its rows are not computed at all
  c->Tf = c->T - 1;
  c->dh = d.dim / d.n_heads;
  c->r = d.rank;
  check(d.precision == ZO_PREC_FP16 || d.precision == ZO_PREC_BF16 || d.precision == ZO_PREC_FP32, ZO_ERR_CONFIG,
        "unknown precision");
  c->bf16 = d.precision == ZO_PREC_BF16;
  c->real32 = d.precision == ZO_PREC_FP32;
  if (c->real32) {
    check(d.rank <= 8, ZO_ERR_CONFIG, "real32 scorer supports rank <= 8");
    check(c->dh <= 128, ZO_ERR_CONFIG, "real32 scorer supports head dim <= 128");
    check(d.estimator != ZO_EST_DENSE, ZO_ERR_CONFIG, "real32 scorer: dense_mezo runs the 16-bit materialising loop");
  }
  check(d.scope == ZO_SCOPE_LORA_ONLY || d.scope == ZO_SCOPE_FULL, ZO_ERR_CONFIG, "unknown scope");
  check(d.estimator == ZO_EST_LOZO || d.estimator == ZO_EST_FACTORIZED || d.estimator == ZO_EST_DENSE, ZO_ERR_CONFIG,
        "unknown estimator");
  c->dense = d.estimator == ZO_EST_DENSE;
  // dense_mezo perturbs every parameter (scope ignored, zo_engine.py:486-488): the 1-D params
  // take the full-scope direction machinery
  c->full_scope = d.scope == ZO_SCOPE_FULL || c->dense;
  check(d.arch == ZO_ARCH_ZOSERVE || d.arch == ZO_ARCH_OPT, ZO_ERR_CONFIG, "unknown architecture");
  c->opt = d.arch == ZO_ARCH_OPT;
  if (c->opt) check(d.max_pos >= c->T, ZO_ERR_DIMENSION, "max_pos shorter than the sequence");
  // rank <= 8: fused fp32 extension dots carried as (hi, lo, hi) 16-bit columns; above:
  // one 16-bit column per rank from the tensor-core extension GEMM
  c->ext_terms = d.rank <= 8 ? 3 : 1;
  c->ext_used = c->ext_terms * d.rank;
  c->KE = (int)ceil_div(c->ext_used, 64) * 64;
  for (auto& e : c->ev) ZO_CUDA_TRY(cudaEventCreate(&e));
  c->flags = c->mem.get<unsigned>(4);

  // registry in sorted layer-id order (matrix_ids, model.py:120-121)
  const int64_t D = d.dim;
  std::vector<Matrix> ms;
  auto add = [&](const std::string& lid, int kind, int layer, int64_t m, int64_t n) {
    Matrix x;
    x.lid = lid;
    x.kind = kind;
    x.layer = layer;
    x.m = m;
    x.n = n;
    x.lid_hash = fnv(lid.data(), lid.size(), FNV0);
    ms.push_back(x);
  };
  add("embed", K_EMBED, -1, d.vocab, D);
  if (c->opt) add("pos_embed", K_POS, -1, (int64_t)d.max_pos + 2, D);
  for (int l = 0; l < d.n_layers; ++l) {
    const std::string p = "blk" + std::to_string(l) + ".";
    add(p + "qkv", K_QKV, l, D, 3 * D);
    add(p + "attn_out", K_OUT, l, D, D);
    add(p + "ff_up", K_UP, l, D, 4 * D);
    add(p + "ff_down", K_DOWN, l, 4 * D, D);
  }
  std::sort(ms.begin(), ms.end(), [](const Matrix& a, const Matrix& b) { return a.lid < b.lid; });
  for (auto& m : ms) {
    check(d.estimator != ZO_EST_LOZO || d.rank <= std::min(m.m, m.n), ZO_ERR_CONFIG,
          "rank " + std::to_string(d.rank) + " exceeds min dim of " + m.lid);
    m.u_off = c->su;
    m.v_off = c->sv;
    c->su += m.m * d.rank;
    c->sv += m.n * d.rank;
  }
  c->mats = ms;
  c->i_qkv.assign(d.n_layers, -1);
  c->i_out.assign(d.n_layers, -1);
  c->i_up.assign(d.n_layers, -1);
  c->i_down.assign(d.n_layers, -1);
  for (size_t i = 0; i < c->mats.size(); ++i) {
    Matrix& m = c->mats[i];
    if (m.kind == K_EMBED) c->i_embed = (int)i;
    if (m.kind == K_POS) c->i_pos = (int)i;
    if (m.kind == K_QKV) c->i_qkv[m.layer] = (int)i;
    if (m.kind == K_OUT) c->i_out[m.layer] = (int)i;
    if (m.kind == K_UP) c->i_up[m.layer] = (int)i;
    if (m.kind == K_DOWN) c->i_down[m.layer] = (int)i;
  }
  // weights
  for (auto& m : c->mats) {
    m.W64 = c->mem.get<double>((size_t)(m.m * m.n));
    if (m.kind == K_EMBED) {
      m.ldw = (int)m.n;
      m.W16 = c->mem.get<uint16_t>((size_t)(m.m * m.n));
    } else if (m.kind == K_POS) {  // read as float64 by the embedding gather: no 16-bit copy
      m.ldw = (int)m.n;
      m.W16 = nullptr;
    } else {
      m.ldw = (int)(m.m + c->KE);
      m.W16 = c->mem.get<uint16_t>((size_t)(m.n * m.ldw));
    }
  }
  if (c->real32) {
    // 3xTF32 split operands: 12 bytes per weight beside the float64 master
    double need = 0;
    for (auto& m : c->mats)
      if (m.kind != K_POS) need += 12.0 * (double)m.m * (double)m.n;
    size_t free_b = 0, total_b = 0;
    ZO_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    check(need + 4e9 < (double)free_b, ZO_ERR_CONFIG,
          "real32: the 3xTF32 split weights (" + std::to_string((long long)(need / 1e9)) +
              " GB) do not fit beside the float64 master; use fp16/bf16 at this size");
    for (auto& m : c->mats) {
      if (m.kind == K_POS) continue;
      if (m.kind == K_EMBED) {
        m.ldk = (int)ceil_div(3 * m.n, 32) * 32;
        m.W32S = c->mem.get<float>((size_t)m.m * m.ldk);
      } else {
        m.ldk = (int)ceil_div(3 * m.m + 3 * d.rank, 32) * 32;
        m.W32S = c->mem.get<float>((size_t)m.n * m.ldk);
      }
    }
  }
  // slots
  c->U = c->mem.get<double>(c->su);
  c->A = c->mem.get<double>(c->su);
  c->V = c->mem.get<double>(c->sv);
  c->Pp = c->mem.get<float>(c->su);
  c->Pm = c->mem.get<float>(c->su);
  c->V32 = c->mem.get<float>(c->sv);
  if (c->dense) {
    for (auto& m : c->mats) {
      m.z_off = c->szm;
      c->szm += m.m * m.n;
    }
    size_t free_b = 0, total_b = 0;
    ZO_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    check((double)c->szm * 8.0 + 4e9 < (double)free_b, ZO_ERR_CONFIG,
          "dense_mezo: the dense direction arena (" + std::to_string(c->szm * 8 / 1000000000) +
              " GB) does not fit beside the float64 master");
    c->ZM = c->mem.get<double>(c->szm);
  }
  // 1-D params (identity at init, model.py:100-107; OPT biases zero), sorted ids
  {
    std::vector<std::pair<std::string, int64_t>> vs;
    for (int l = 0; l < d.n_layers; ++l) {
      const std::string p = "blk" + std::to_string(l) + ".";
      for (const char* w : {"ln1.scale", "ln1.shift", "ln2.scale", "ln2.shift"}) vs.push_back({p + w, D});
      if (c->opt) {
        vs.push_back({p + "qkv.bias", 3 * D});
        vs.push_back({p + "attn_out.bias", D});
        vs.push_back({p + "ff_up.bias", 4 * D});
        vs.push_back({p + "ff_down.bias", D});
      }
    }
    vs.push_back({"ln_f.scale", D});
    vs.push_back({"ln_f.shift", D});
    std::sort(vs.begin(), vs.end());
    for (auto& v : vs) {
      c->vids.push_back(v.first);
      c->voff.push_back(c->nvt);
      c->vlen.push_back(v.second);
      c->nvt += v.second;
    }
  }
  c->nv = (int)c->vids.size();
  const size_t nvd = (size_t)c->nvt;
  c->VEC64 = c->mem.get<double>(nvd);
  c->VEC32 = c->mem.get<float>(2 * nvd);
  {
    std::vector<double> init(nvd, 0.0);
    for (int v = 0; v < c->nv; ++v)
      if (c->vids[v].size() >= 6 && c->vids[v].compare(c->vids[v].size() - 6, 6, ".scale") == 0)
        std::fill(init.begin() + c->voff[v], init.begin() + c->voff[v] + c->vlen[v], 1.0);
    ZO_CUDA_TRY(cudaMemcpy(c->VEC64, init.data(), nvd * 8, cudaMemcpyHostToDevice));
    launch_vec_probe(c->VEC64, nullptr, (int64_t)nvd, 0.0, c->VEC32, nullptr);
    ZO_CUDA_TRY(cudaDeviceSynchronize());
  }
  auto vptr = [&](const std::string& id) {
    const int v = (int)(std::lower_bound(c->vids.begin(), c->vids.end(), id) - c->vids.begin());
    return c->VEC32 + c->voff[v];
  };
  for (int l = 0; l < d.n_layers; ++l) {
    const std::string p = "blk" + std::to_string(l) + ".";
    c->ln1g.push_back(vptr(p + "ln1.scale"));
    c->ln1b.push_back(vptr(p + "ln1.shift"));
    c->ln2g.push_back(vptr(p + "ln2.scale"));
    c->ln2b.push_back(vptr(p + "ln2.shift"));
    c->bqkv.push_back(c->opt ? vptr(p + "qkv.bias") : nullptr);
    c->bout.push_back(c->opt ? vptr(p + "attn_out.bias") : nullptr);
    c->bup.push_back(c->opt ? vptr(p + "ff_up.bias") : nullptr);
    c->bdown.push_back(c->opt ? vptr(p + "ff_down.bias") : nullptr);
  }
  c->lnfg = vptr("ln_f.scale");
  c->lnfb = vptr("ln_f.shift");
  if (c->full_scope) {
    c->VZ = c->mem.get<double>(nvd);
    c->vstride = (long)nvd;
  }
  // activations
  c->Mmax = 2 * d.max_batch * c->T;
  c->Mpad = (int)ceil_div(c->Mmax, 128) * 128;
  c->Smax = 2 * d.max_batch * d.opt_len;
  c->Spad = (int)ceil_div(c->Smax, 128) * 128;
  c->ldl = (int)ceil_div(d.vocab, 4) * 4;
  c->x32 = c->mem.get<float>((size_t)c->Mpad * D);
  c->hA = c->mem.get<uint16_t>((size_t)c->Mpad * (D + c->KE));
  c->qkv = c->mem.get<uint16_t>((size_t)c->Mpad * 3 * D);
  c->ctxA = c->mem.get<uint16_t>((size_t)c->Mpad * (D + c->KE));
  c->gA = c->mem.get<uint16_t>((size_t)c->Mpad * (4 * D + c->KE));
  c->xs16 = c->mem.get<uint16_t>((size_t)c->Spad * D);
  c->hS = c->mem.get<uint16_t>((size_t)c->Spad * (D + c->KE));
  c->gS = c->mem.get<uint16_t>((size_t)c->Spad * (4 * D + c->KE));
  c->x32S = c->mem.get<float>((size_t)c->Spad * D);
  if (c->real32) {
    c->lda32 = (int)ceil_div(12 * D + 3 * d.rank, 32) * 32;
    c->a32 = c->mem.get<float>((size_t)c->Mpad * c->lda32);
    c->f32a = c->mem.get<float>((size_t)c->Mpad * 4 * D);
    c->ctx32 = c->mem.get<float>((size_t)c->Mpad * D);
  }

  c->xs32 = c->mem.get<float>((size_t)c->Smax * D);
  c->z = c->mem.get<float>((size_t)c->Smax * d.rank);
  c->logits = c->mem.get<float>((size_t)c->Smax * c->ldl);
  c->loss_ws = c->mem.get<float>(loss_ws_floats(c->Smax, d.vocab));
  c->loss_cnt = c->mem.get<unsigned>(2 * (size_t)c->Smax);
  c->nll = c->mem.get<double>(2 * std::max(d.max_batch, 4096));
  c->nll_bl = c->mem.get<double>(d.max_batch);
  c->out4 = c->mem.get<double>(4);
  c->abort_flag = c->mem.get<unsigned>(1);
  c->tok = c->mem.get<int32_t>((size_t)d.max_batch * c->T);
  c->gold = c->mem.get<int32_t>((size_t)2 * d.max_batch * d.opt_len);
  c->d_step = c->mem.get<uint64_t>(1);
  c->d_base = c->mem.get<uint64_t>(1);
  c->sk_ws = c->mem.get<float>(gemm_sk_ws_floats(c->num_sms));
  c->sk_flags = c->mem.get<unsigned>(c->num_sms + 1);
  if (env_streamk_off()) c->streamk = false;
  c->fused_ext = d.rank <= 8;
  c->tpart_tiles = std::max((int)ceil_div(4 * D, 64), d.n_heads);
  if (c->fused_ext) c->tpart = c->mem.get<float>((size_t)c->tpart_tiles * c->Mpad * d.rank);
  else {
    c->P16T = c->mem.get<uint16_t>((size_t)2 * c->su);
    std::vector<int64_t> tab;
    for (const auto& m : c->mats) {
      if (m.kind == K_EMBED || m.kind == K_POS) continue;
      tab.insert(tab.end(), {(int64_t)c->p16t_tiles, m.u_off, m.m});
      c->p16t_tiles += (int)ceil_div(m.m, 32);
    }
    c->p16t_n = (int)(tab.size() / 3);
    c->p16t_tab = c->mem.get<int64_t>(tab.size() + 1);
    if (!tab.empty())
      ZO_CUDA_TRY(cudaMemcpy(c->p16t_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
    c->xws = c->mem.get<float>((size_t)c->num_sms * c->Mpad * d.rank);
  }
  // positional table: pos_encoding(T, d) (model.py:128-136), float64 -> float32
  {
    std::vector<float> pe((size_t)c->T * d.dim);
    for (int t = 0; t < c->T; ++t)
      for (int j = 0; j < d.dim; ++j) {
        const double ang = (double)t / std::pow(10000.0, (2.0 * (j / 2)) / (double)d.dim);
        pe[(size_t)t * d.dim + j] = (float)((j % 2 == 0) ? std::sin(ang) : std::cos(ang));
      }
    c->pe = c->mem.get<float>(pe.size());
    ZO_CUDA_TRY(cudaMemcpy(c->pe, pe.data(), pe.size() * 4, cudaMemcpyHostToDevice));
  }
  ZO_CUDA_TRY(cudaMallocHost(&c->h_tok, (size_t)d.max_batch * c->T * 4));
  ZO_CUDA_TRY(cudaMallocHost(&c->h_gold, (size_t)2 * d.max_batch * d.opt_len * 4));
  ZO_CUDA_TRY(cudaMallocHost(&c->h_out4, 4 * 8));
  ZO_CUDA_TRY(cudaMallocHost(&c->h_step, 8));
  // sampler plans: U (step), V (window start for lozo, step for factorized)
  for (auto& m : c->mats) {
    StreamDesc su{};
    su.lid_hash = m.lid_hash;
    su.role = 0;
    su.step_mode = STEP_CURRENT;
    su.n = (uint64_t)(m.m * d.rank);
    su.out_off = (uint64_t)m.u_off;
    su.scale = 1.0;
    c->streamsU.push_back(su);
    StreamDesc sv = su;
    sv.role = 1;
    sv.step_mode = d.estimator == ZO_EST_LOZO ? STEP_WINDOW : STEP_CURRENT;
    sv.n = (uint64_t)(m.n * d.rank);
    sv.out_off = (uint64_t)m.v_off;
    c->streamsV.push_back(sv);
  }
  // the direction plans emit by copy (one Philox pass per sample)
  build_sampler_plan(c.get(), c->planU, c->streamsU, true);
  build_sampler_plan(c.get(), c->planV, c->streamsV, true);
  if (c->dense) {
    // dense_direction(seed, step, lid, (m, n)) = sample_gaussian(key DENSE_Z, m, n) row-major
    for (auto& m : c->mats) {
      StreamDesc sz{};
      sz.lid_hash = m.lid_hash;
      sz.role = 2;  // Role.DENSE_Z
      sz.step_mode = STEP_CURRENT;
      sz.n = (uint64_t)(m.m * m.n);
      sz.out_off = (uint64_t)m.z_off;
      sz.scale = 1.0;
      c->streamsZM.push_back(sz);
    }
    build_sampler_plan(c.get(), c->planZM, c->streamsZM);
  }
  if (c->full_scope) {
    // dense_direction(seed, step, vid, (dim,)) = gaussian_vector (zo_engine.py:194-198)
    for (int v = 0; v < c->nv; ++v) {
      StreamDesc sz{};
      sz.lid_hash = fnv(c->vids[v].data(), c->vids[v].size(), FNV0);
      sz.role = 2;  // Role.DENSE_Z
      sz.step_mode = STEP_CURRENT;
      sz.n = (uint64_t)c->vlen[v];
      sz.out_off = (uint64_t)c->voff[v];
      sz.scale = 1.0;
      c->streamsZ.push_back(sz);
    }
    build_sampler_plan(c.get(), c->planZ, c->streamsZ);
  }
  ZO_CUDA_TRY(cudaDeviceSynchronize());
  *out = c.release();
  return ZO_OK;
  ZO_API_END
}

int zo_destroy(zo_ctx* c) {
  ZO_API_BEGIN
  if (c) {
    cudaStreamSynchronize(c->st);
    delete c;
  }
  return ZO_OK;
  ZO_API_END
}

int zo_set_stream(zo_ctx* c, void* s) {
  c->st = static_cast<cudaStream_t>(s);
  return ZO_OK;
}

int zo_synchronize(zo_ctx* c) {
  ZO_API_BEGIN
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

int zo_num_matrices(const zo_ctx* c) { return (int)c->mats.size(); }

int zo_matrix_info(const zo_ctx* c, int i, char* lid, int cap, int64_t* rows, int64_t* cols) {
  if (i < 0 || i >= (int)c->mats.size()) return ZO_ERR_INPUT;
  const Matrix& m = c->mats[i];
  if (lid && cap > 0) {
    std::strncpy(lid, m.lid.c_str(), cap - 1);
    lid[cap - 1] = 0;
  }
  if (rows) *rows = m.m;
  if (cols) *cols = m.n;
  return ZO_OK;
}

int zo_device_bytes(const zo_ctx* c, uint64_t* bytes) {
  *bytes = c->mem.bytes;
  return ZO_OK;
}

int zo_init_params(zo_ctx* c, uint64_t init_seed, double init_scale) {
  ZO_API_BEGIN
  // one plan per matrix (bounded chunk arrays), Role.INIT at step 0 (model.py:94-96)
  for (auto& m : c->mats) {
    std::vector<StreamDesc> sd(1);
    sd[0].lid_hash = m.lid_hash;
    sd[0].role = 4;
    sd[0].step_mode = STEP_FIXED;
    sd[0].fixed_step = 0;
    sd[0].n = (uint64_t)(m.m * m.n);
    sd[0].out_off = 0;
    sd[0].scale = init_scale;
    sd[0].apply_scale = 1;
    sd[0].seed_override = 1;
    sd[0].seed_value = init_seed;
    DevAlloc tmp;
    SamplerPlan P;
    // temporary plan (freed after the matrix is done)
    int64_t nch = (int64_t)sampler_chunks_for(sd[0].n);
    sd[0].chunk_begin = 0;
    sd[0].n_chunks = (uint64_t)nch;
    P.S = 1;
    P.C = nch;
    P.d_streams = tmp.get<StreamDesc>(1);
    P.d_chunk_stream = tmp.get<uint32_t>(nch);  // zeros: every chunk belongs to stream 0
    P.d_keys = tmp.get<uint64_t>(2);
    P.d_spec = tmp.get<uint64_t>(nch);
    P.d_exit = tmp.get<uint64_t>(nch);
    P.d_count = tmp.get<uint32_t>(nch);
    P.d_offset = tmp.get<uint64_t>(nch);
    P.d_flags = c->flags;
    ZO_CUDA_TRY(cudaMemcpyAsync(P.d_streams, sd.data(), sizeof(StreamDesc), cudaMemcpyHostToDevice, c->st));
    sampler_launch(P, init_seed, c->d_step, 1, m.W64, c->st);
    refresh_shadow(c, m);
    if (c->master32 && has_master32(m)) narrow_master(c, m);
    ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  }
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

int zo_upload_matrix(zo_ctx* c, const char* lid, const double* host, int64_t rows, int64_t cols) {
  ZO_API_BEGIN
  Matrix& m = find(c, lid);
  check(rows == m.m && cols == m.n, ZO_ERR_DIMENSION, "matrix shape mismatch for " + m.lid);
  ZO_CUDA_TRY(cudaMemcpyAsync(m.W64, host, (size_t)(rows * cols) * 8, cudaMemcpyHostToDevice, c->st));
  refresh_shadow(c, m);
  if (c->master32 && has_master32(m)) narrow_master(c, m);
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

int zo_download_matrix(zo_ctx* c, const char* lid, double* host, int64_t rows, int64_t cols) {
  ZO_API_BEGIN
  Matrix& m = find(c, lid);
  check(rows == m.m && cols == m.n, ZO_ERR_DIMENSION, "matrix shape mismatch for " + m.lid);
  with_master64(c, m, [&] {
    ZO_CUDA_TRY(cudaMemcpyAsync(host, m.W64, (size_t)(rows * cols) * 8, cudaMemcpyDeviceToHost, c->st));
  });
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

static int vector_index(const zo_ctx* c, const char* lid) {
  auto it = std::lower_bound(c->vids.begin(), c->vids.end(), std::string(lid));
  check(it != c->vids.end() && *it == lid, ZO_ERR_INPUT, std::string("unknown vector id ") + lid);
  return (int)(it - c->vids.begin());
}

int zo_upload_vector(zo_ctx* c, const char* lid, const double* host, int64_t n) {
  ZO_API_BEGIN
  const int v = vector_index(c, lid);
  check(n == c->vlen[v], ZO_ERR_DIMENSION, std::string("vector length mismatch for ") + lid);
  const size_t nvd = (size_t)c->nvt, o = (size_t)c->voff[v];
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaMemcpy(c->VEC64 + o, host, n * 8, cudaMemcpyHostToDevice));
  std::vector<float> f(n);
  for (int64_t i = 0; i < n; ++i) f[i] = (float)host[i];
  ZO_CUDA_TRY(cudaMemcpy(c->VEC32 + o, f.data(), n * 4, cudaMemcpyHostToDevice));
  ZO_CUDA_TRY(cudaMemcpy(c->VEC32 + nvd + o, f.data(), n * 4, cudaMemcpyHostToDevice));
  return ZO_OK;
  ZO_API_END
}

int zo_download_vector(zo_ctx* c, const char* lid, double* host, int64_t n) {
  ZO_API_BEGIN
  const int v = vector_index(c, lid);
  check(n == c->vlen[v], ZO_ERR_DIMENSION, std::string("vector length mismatch for ") + lid);
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaMemcpy(host, c->VEC64 + c->voff[v], n * 8, cudaMemcpyDeviceToHost));
  return ZO_OK;
  ZO_API_END
}

int zo_sample_u(zo_ctx* c, uint64_t seed, uint64_t step) {
  ZO_API_BEGIN
  set_step(c, step);
  sampler_launch(c->planU, seed, c->d_step, 1, c->U, c->st);
  sample_z(c, seed);
  return ZO_OK;
  ZO_API_END
}

int zo_sample_v(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu) {
  ZO_API_BEGIN
  check(nu >= 1, ZO_ERR_CONFIG, "nu must be >= 1");
  // unfolded window mass must be folded before V changes (zo_engine.py:395-398)
  if (c->d.estimator == ZO_EST_LOZO && c->a_dirty) fold_all(c);
  set_step(c, step);
  sampler_launch(c->planV, seed, c->d_step, (uint32_t)nu, c->V, c->st);
  write_vext_all(c);
  c->v_window = c->d.estimator == ZO_EST_LOZO ? (int64_t)((step / (uint64_t)nu) * (uint64_t)nu) : (int64_t)step;
  return ZO_OK;
  ZO_API_END
}

int zo_sample_stream(zo_ctx* c, uint64_t seed, uint64_t step, uint64_t lid_hash, int32_t role, int64_t n,
                     double* host_out) {
  ZO_API_BEGIN
  check(n >= 1, ZO_ERR_DIMENSION, "gaussian sample needs n >= 1");
  // ctx may be NULL: sample on the current device / default stream
  cudaStream_t st = c ? c->st : (cudaStream_t)0;
  DevAlloc tmp;
  unsigned* flags = c ? c->flags : tmp.get<unsigned>(4);
  uint64_t* dstep = c ? c->d_step : tmp.get<uint64_t>(1);
  std::vector<StreamDesc> sd(1);
  sd[0].lid_hash = lid_hash;
  sd[0].role = (uint32_t)role;
  sd[0].step_mode = STEP_FIXED;
  sd[0].fixed_step = step;
  sd[0].n = (uint64_t)n;
  sd[0].scale = 1.0;
  SamplerPlan P;
  int64_t nch = (int64_t)sampler_chunks_for((uint64_t)n);
  sd[0].n_chunks = (uint64_t)nch;
  P.S = 1;
  P.C = nch;
  P.d_streams = tmp.get<StreamDesc>(1);
  P.d_chunk_stream = tmp.get<uint32_t>(nch);
  P.d_keys = tmp.get<uint64_t>(2);
  P.d_spec = tmp.get<uint64_t>(nch);
  P.d_exit = tmp.get<uint64_t>(nch);
  P.d_count = tmp.get<uint32_t>(nch);
  P.d_offset = tmp.get<uint64_t>(nch);
  P.d_flags = flags;
  double* out = tmp.get<double>((size_t)n);
  ZO_CUDA_TRY(cudaMemcpyAsync(P.d_streams, sd.data(), sizeof(StreamDesc), cudaMemcpyHostToDevice, st));
  sampler_launch(P, seed, dstep, 1, out, st);
  ZO_CUDA_TRY(cudaMemcpyAsync(host_out, out, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  ZO_CUDA_TRY(cudaStreamSynchronize(st));
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

int zo_slot_count(const zo_ctx* c, int32_t which, int64_t* count) {
  if (which < 0 || which > 4 || (which == 3 && !c->full_scope) || (which == 4 && !c->dense)) return ZO_ERR_INPUT;
  *count = which == 4 ? c->szm : which == 3 ? c->nvt : which == 1 ? c->sv : c->su;
  return ZO_OK;
}

static double* slot_ptr(zo_ctx* c, int which) {
  return which == 0 ? c->U : which == 1 ? c->V : which == 2 ? c->A : which == 3 ? c->VZ : c->ZM;
}
static int64_t slot_size(const zo_ctx* c, int which) {
  return which == 4 ? c->szm : which == 3 ? c->nvt : which == 1 ? c->sv : c->su;
}

int zo_get_slot(zo_ctx* c, int32_t which, double* host, int64_t count) {
  ZO_API_BEGIN
  check(which >= 0 && which <= 4 && (which != 3 || c->full_scope) && (which != 4 || c->dense), ZO_ERR_INPUT,
        "bad slot id");
  check(count == slot_size(c, which), ZO_ERR_DIMENSION, "slot arena size mismatch");
  ZO_CUDA_TRY(cudaMemcpyAsync(host, slot_ptr(c, which), (size_t)count * 8, cudaMemcpyDeviceToHost, c->st));
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

// Snapshot the U (0) or V (1) arena into pinned host ring slot `slot` without blocking the
// step stream: a device-to-device copy in stream order (the next step's sampler may then
// overwrite the arena), then the device-to-host copy on a side stream that overlaps the next
// step.  zo_slot_snapshot_wait blocks until that slot's copy has landed and returns it.
int zo_slot_snapshot(zo_ctx* c, int32_t which, int32_t slot) {
  ZO_API_BEGIN
  check(which == 0 || which == 1, ZO_ERR_INPUT, "snapshots cover the U and V arenas");
  check(slot >= 0 && slot < zo_ctx::SNAP_RING, ZO_ERR_INPUT, "snapshot slot out of range");
  const size_t n = which == 1 ? (size_t)c->sv : (size_t)c->su;
  if (!c->snap_st) ZO_CUDA_TRY(cudaStreamCreateWithFlags(&c->snap_st, cudaStreamNonBlocking));
  if (!c->snap_dev[which]) c->snap_dev[which] = c->mem.get<double>(n);
  if (!c->snap_host[which][slot]) {
    // the whole ring at once (pinned allocations take milliseconds: none inside a run's
    // steady state, e.g. at the first window boundary of a timed span)
    for (int k = 0; k < zo_ctx::SNAP_RING; ++k) {
      if (c->snap_host[which][k]) continue;
      ZO_CUDA_TRY(cudaMallocHost(&c->snap_host[which][k], n * 8));
      ZO_CUDA_TRY(cudaEventCreateWithFlags(&c->snap_ready[which][k], cudaEventDisableTiming));
      ZO_CUDA_TRY(cudaEventCreateWithFlags(&c->snap_done[which][k], cudaEventDisableTiming));
    }
  }
  // the previous D2H out of the device copy must be done before it is overwritten, and this
  // host slot's previous copy must have been consumed (the caller waited on it)
  if (c->snap_last[which]) ZO_CUDA_TRY(cudaStreamWaitEvent(c->st, c->snap_last[which], 0));
  ZO_CUDA_TRY(cudaMemcpyAsync(c->snap_dev[which], slot_ptr(c, which), n * 8, cudaMemcpyDeviceToDevice, c->st));
  ZO_CUDA_TRY(cudaEventRecord(c->snap_ready[which][slot], c->st));
  ZO_CUDA_TRY(cudaStreamWaitEvent(c->snap_st, c->snap_ready[which][slot], 0));
  ZO_CUDA_TRY(cudaMemcpyAsync(c->snap_host[which][slot], c->snap_dev[which], n * 8, cudaMemcpyDeviceToHost,
                              c->snap_st));
  ZO_CUDA_TRY(cudaEventRecord(c->snap_done[which][slot], c->snap_st));
  c->snap_last[which] = c->snap_done[which][slot];
  c->snap_taken[which][slot] = true;
  return ZO_OK;
  ZO_API_END
}

int zo_slot_snapshot_wait(zo_ctx* c, int32_t which, int32_t slot, const double** host) {
  ZO_API_BEGIN
  check((which == 0 || which == 1) && slot >= 0 && slot < zo_ctx::SNAP_RING && c->snap_taken[which][slot],
        ZO_ERR_INPUT, "no such snapshot");
  ZO_CUDA_TRY(cudaEventSynchronize(c->snap_done[which][slot]));
  *host = c->snap_host[which][slot];
  return ZO_OK;
  ZO_API_END
}

int zo_set_slot(zo_ctx* c, int32_t which, const double* host, int64_t count) {
  ZO_API_BEGIN
  check(which >= 0 && which <= 2, ZO_ERR_INPUT, "bad slot id");
  check(count == (which == 1 ? c->sv : c->su), ZO_ERR_DIMENSION, "slot arena size mismatch");
  ZO_CUDA_TRY(cudaMemcpyAsync(slot_ptr(c, which), host, (size_t)count * 8, cudaMemcpyHostToDevice, c->st));
  // host directions: refresh the tensor update's 16-bit copies the sampler would have written
  if (which == 0 && c->planU.out16) launch_shadow(c->U, c->su, c->U16, c->bf16, c->st);
  if (which == 1 && c->planV.out16) launch_shadow(c->V, c->sv, c->V16, c->bf16, c->st);
  if (which == 1) {
    write_vext_all(c);
    // a host V carries no window key: the next step resamples V (folding A with THIS V
    // first) unless the caller declares the window with zo_set_window
    c->v_window = -2;
  }
  if (which == 2) {
    bool nz = false;
    for (int64_t i = 0; i < count && !nz; ++i) nz = host[i] != 0.0;
    c->a_dirty = nz;  // uploaded window mass must be folded before V changes
  }
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

int zo_set_update_mode(zo_ctx* c, int32_t mode) {
  ZO_API_BEGIN
  check(mode == 0 || mode == 1, ZO_ERR_CONFIG, "update mode must be 0 (exact) or 1 (tensor)");
  if (mode == 1) {
    check(c->d.estimator == ZO_EST_FACTORIZED, ZO_ERR_CONFIG, "the tensor-core dense update serves factorized_sqrt_r");
    check(c->r >= 16 && c->r % 16 == 0, ZO_ERR_CONFIG, "the tensor-core dense update needs rank >= 16, multiple of 16");
    check(!c->real32, ZO_ERR_CONFIG, "real32 keeps the exact float64 update");
    if (!c->U16) {
      // + 256 rows of padding: an update GEMM's A-operand tensor map spans the matrix's rows
      // rounded up to the 128-row tile, so the last matrix's box reads past its slice
      c->U16 = c->mem.get<uint16_t>((size_t)c->su + (size_t)256 * c->r);
      c->V16 = c->mem.get<uint16_t>((size_t)c->sv + (size_t)256 * c->r);
    }
  }
  // tensor mode: the direction sampler writes the update's 16-bit U / V operands as it emits
  c->planU.out16 = mode == 1 ? c->U16 : nullptr;
  c->planV.out16 = mode == 1 ? c->V16 : nullptr;
  c->planU.out16_bf16 = c->planV.out16_bf16 = c->bf16;
  if ((mode == 1) != c->master32) {
    if (!c->conv_tmp) c->conv_tmp = c->mem.get<float>(CONV_CHUNK);
    for (auto& m : c->mats) {
      if (!has_master32(m)) continue;
      if (mode == 1) narrow_master(c, m);
      else widen_master(c, m);
    }
    c->master32 = mode == 1;
    ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  }
  c->fast_update = mode == 1;
  c->upd_plans.clear();
  c->drop_graphs();  // the captured step graphs hold the old update
  return ZO_OK;
  ZO_API_END
}

int zo_set_schedule(zo_ctx* c, int32_t row_invariant) {
  ZO_API_BEGIN
  check(row_invariant == 0 || row_invariant == 1, ZO_ERR_CONFIG, "schedule must be 0 (fastest) or 1 (row-invariant)");
  const bool sk = row_invariant == 0 && !env_streamk_off();
  if (sk != c->streamk) {
    ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
    c->streamk = sk;
    c->plans.clear();        // GEMM plans carry the stream-K split
    c->drop_graphs();        // the captured step graphs hold the old plans
  }
  return ZO_OK;
  ZO_API_END
}

int zo_set_window(zo_ctx* c, int64_t window_start) {
  ZO_API_BEGIN
  check(window_start >= -1, ZO_ERR_INPUT, "window start must be >= -1");
  c->v_window = window_start;
  return ZO_OK;
  ZO_API_END
}

int zo_sampler_flags(zo_ctx* c, uint32_t flags[3]) {
  ZO_API_BEGIN
  unsigned f[4];
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaMemcpy(f, c->flags, sizeof(f), cudaMemcpyDeviceToHost));
  flags[0] = f[0];
  flags[1] = f[1];
  flags[2] = f[2];
  return ZO_OK;
  ZO_API_END
}

int zo_prepare_probe(zo_ctx* c, double eps, int32_t sign_mode) {
  ZO_API_BEGIN
  // sign_mode 0: P+- = A +- eps*scale*U (probe pair); 1: P = A (no probe, sign 0)
  const double scale = c->d.estimator == ZO_EST_FACTORIZED ? 1.0 / std::sqrt((double)c->r) : 1.0;
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  launch_prep_probe(lozo ? c->A : nullptr, c->U, c->su, sign_mode == 0 ? eps : 0.0, scale, c->Pp, c->Pm, c->st);
  vec_probe(c, sign_mode == 0 ? eps : 0.0);
  c->probe_eps = eps;
  c->probe_scale = scale;
  return ZO_OK;
  ZO_API_END
}

int zo_score(zo_ctx* c, const int32_t* tokens, const int32_t* gold, int32_t B, int32_t nsign, double* nll_out) {
  ZO_API_BEGIN
  check(nsign == 1 || nsign == 2, ZO_ERR_INPUT, "nsign must be 1 or 2");
  check(B >= 1 && B <= c->d.max_batch, ZO_ERR_DIMENSION, "batch size out of range");
  stage_batch(c, tokens, gold, B, nsign);
  do_score(c, B, nsign);
  if (nll_out) {
    ZO_CUDA_TRY(cudaMemcpyAsync(nll_out, c->nll, (size_t)nsign * B * 8, cudaMemcpyDeviceToHost, c->st));
    ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  }
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

int zo_score_options(zo_ctx* c, const int32_t* tokens, const int32_t* options, int32_t n_opt, int32_t B,
                     double* nll_out) {
  ZO_API_BEGIN
  check(c->d.opt_len == 1, ZO_ERR_CONFIG, "one-forward option scoring needs single-token options");
  check(c->fused_ext && !c->real32, ZO_ERR_CONFIG, "one-forward option scoring: rank <= 8, 16-bit modes");
  check(n_opt >= 1 && B >= 1 && B <= c->d.max_batch, ZO_ERR_DIMENSION, "bad option count / batch size");
  std::vector<int32_t> gold((size_t)B);
  for (int32_t j = 0; j < n_opt; ++j) {
    std::fill(gold.begin(), gold.end(), options[j]);
    if (j == 0) {
      stage_batch(c, tokens, gold.data(), B, 1);
      do_score(c, B, 1);  // logits of the scored rows stay in c->logits
    } else {
      check(options[j] >= 0 && options[j] < c->d.vocab, ZO_ERR_INPUT, "gold token id out of range");
      ZO_CUDA_TRY(cudaStreamSynchronize(c->st));  // the pinned gold staging is reused
      std::memcpy(c->h_gold, gold.data(), (size_t)B * 4);
      std::memcpy(c->h_gold + B, gold.data(), (size_t)B * 4);
      ZO_CUDA_TRY(cudaMemcpyAsync(c->gold, c->h_gold, (size_t)2 * B * 4, cudaMemcpyHostToDevice, c->st));
      const Matrix& e = c->mats[c->i_embed];
      launch_loss(c->logits, c->ldl, c->d.vocab, c->z, c->r, c->Pp + e.u_off, c->Pm + e.u_off, c->gold, B, 1,
                  c->loss_ws, c->loss_cnt, c->nll, c->st);
    }
    ZO_CUDA_TRY(cudaMemcpyAsync(nll_out + (size_t)j * B, c->nll, (size_t)B * 8, cudaMemcpyDeviceToHost, c->st));
  }
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

int zo_coefficient(zo_ctx* c, int32_t B, double eps, double lr, int32_t divide_by_r, double* out4) {
  ZO_API_BEGIN
  launch_coefficient(c->nll, B, eps, lr, divide_by_r, c->r, c->out4, c->abort_flag, c->st);
  ZO_CUDA_TRY(cudaMemcpyAsync(c->h_out4, c->out4, 32, cudaMemcpyDeviceToHost, c->st));
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  if (out4) std::memcpy(out4, c->h_out4, 32);
  if (!std::isfinite(c->h_out4[0]) || !std::isfinite(c->h_out4[1]))
    throw Error(ZO_ERR_ABORT, "non-finite paired loss; step not applied");
  return ZO_OK;
  ZO_API_END
}

int zo_set_coefficient(zo_ctx* c, const double* out4) {
  ZO_API_BEGIN
  std::memcpy(c->h_out4, out4, 32);
  const unsigned zero = 0;
  ZO_CUDA_TRY(cudaMemcpyAsync(c->out4, c->h_out4, 32, cudaMemcpyHostToDevice, c->st));
  ZO_CUDA_TRY(cudaMemcpyAsync(c->abort_flag, &zero, 4, cudaMemcpyHostToDevice, c->st));
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

int zo_update_u(zo_ctx* c) {
  ZO_API_BEGIN
  launch_update(c->A, c->U, c->su, c->out4, c->abort_flag, c->st);
  c->a_dirty = true;
  return ZO_OK;
  ZO_API_END
}

int zo_fold(zo_ctx* c) {
  ZO_API_BEGIN
  check(!c->master32, ZO_ERR_CONFIG, "fold needs the float64 masters: set update mode 0 first");
  fold_all(c);
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

int zo_update_dense(zo_ctx* c, double lr) {
  ZO_API_BEGIN
  if (c->fast_update) {
    // tensor mode: the installed coefficient (zo_set_coefficient's device copy) drives the
    // fused tcgen05 update, as in a fused step
    launch_dense_update_dev(c, lr, c->out4, nullptr);
    vec_update(c, c->out4, lr, c->abort_flag);
    ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
    return ZO_OK;
  }
  // alpha = -(lr*c) * (1/sqrt(r)) as zo_engine.py:450 computes it (host copy of c)
  const double cc = c->h_out4[2];
  const double alpha = (-(lr * cc)) * (1.0 / std::sqrt((double)c->r));
  for (auto& m : c->mats)
    launch_fold(m.W64, (int)m.m, (int)m.n, c->U + m.u_off, c->V + m.v_off, c->r, alpha, m.W16,
                m.kind == K_EMBED ? (int)m.n : m.ldw, m.kind == K_EMBED ? 0 : 1, c->bf16, c->st);
  vec_update(c, c->out4, lr, c->abort_flag);
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

// full scope: VectorProbe.update with the installed coefficient (zo_engine.py:290-295,
// 412-416) -- the custom-scorer path's complement of zo_update_u
int zo_update_vectors(zo_ctx* c, double lr) {
  ZO_API_BEGIN
  vec_update(c, c->out4, lr, c->abort_flag);
  return ZO_OK;
  ZO_API_END
}

int zo_step(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, double eps, double lr, int32_t divide_by_r,
            const int32_t* tokens, const int32_t* gold, int32_t B, double* out4) {
  ZO_API_BEGIN
  check(!c->dense, ZO_ERR_CONFIG, "dense_mezo has no serving-path form (runtime.py:275-279): use the materialising loop");
  check(nu >= 1, ZO_ERR_CONFIG, "nu must be >= 1");
  check(B >= 1 && B <= c->d.max_batch, ZO_ERR_DIMENSION, "batch size out of range");
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  set_step(c, step);
  stage_batch(c, tokens, gold, B, 1);
  ZO_CUDA_TRY(cudaEventRecord(c->ev[0], c->st));
  const int64_t wstart = lozo ? (int64_t)((step / (uint64_t)nu) * (uint64_t)nu) : (int64_t)step;
  if (!lozo || wstart != c->v_window) {
    // a window start with unfolded mass: fold it first (the reference freezes it
    // into an update slot, zo_engine.py:395-398 -- value-neutral up to rounding)
    if (lozo && c->a_dirty) fold_all(c);
    sampler_launch(c->planV, seed, c->d_step, (uint32_t)nu, c->V, c->st);
    write_vext_all(c);
    c->v_window = wstart;
  }
  ZO_CUDA_TRY(cudaEventRecord(c->ev[1], c->st));
  // U, probes, paired scoring, coefficient and update: the captured step body (bit-identical
  // to eager launches, tests/test_gpu_scorer.py), one graph launch instead of ~370 kernel
  // launches from the host
  graph_body(c, seed, eps, lr, lozo ? divide_by_r : 0, B);
  if (lozo) c->a_dirty = true;
  ZO_CUDA_TRY(cudaEventRecord(c->ev[2], c->st));
  ZO_CUDA_TRY(cudaMemcpyAsync(c->h_out4, c->out4, 32, cudaMemcpyDeviceToHost, c->st));
  ZO_CUDA_TRY(cudaEventRecord(c->ev[3], c->st));
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaGetLastError());
  cudaEventElapsedTime(&c->last_ms[0], c->ev[0], c->ev[1]);
  cudaEventElapsedTime(&c->last_ms[1], c->ev[1], c->ev[2]);
  cudaEventElapsedTime(&c->last_ms[2], c->ev[2], c->ev[3]);
  if (out4) std::memcpy(out4, c->h_out4, 32);
  if (!std::isfinite(c->h_out4[0]) || !std::isfinite(c->h_out4[1]))
    throw Error(ZO_ERR_ABORT, "non-finite paired loss; step not applied");
  return ZO_OK;
  ZO_API_END
}

int zo_last_step_ms(zo_ctx* c, float ms[3]) {
  for (int i = 0; i < 3; ++i) ms[i] = c->last_ms[i];
  return ZO_OK;
}

uint64_t zo_fnv1a64(const void* data, uint64_t nbytes, uint64_t h) { return fnv(data, (size_t)nbytes, h); }

uint64_t zo_digest_chain(const char* const* lids, const double* arena, const int64_t* offsets, const int64_t* counts,
                         int32_t n, uint64_t h) {
  for (int32_t i = 0; i < n; ++i) {
    h = fnv(lids[i], std::strlen(lids[i]), h);
    h = fnv(arena + offsets[i], (size_t)counts[i] * 8, h);
  }
  return h;
}

}  // extern "C"

// Stream-ordered step with device-resident inputs and no host synchronisation
// (tokens_dev [B, T], gold_dev [B, opt_len] int32).  Results stay on the device
// (zo_read_out4); a non-finite loss disarms the update on the device.
// zo_step_score_async = directions + probes + paired scoring (per-example NLLs
// in the ctx); zo_step_apply_async = canonical mean / c / update over B_total
// examples.  Multi-GPU exact mode all-gathers the NLLs between the two.
namespace {
// Step index, device-resident tokens/gold into the ctx, and the window work (fold of the
// unfolded window mass + V resample at a window start): the eager head of every step.
void stage_dev(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, const int32_t* tokens_dev,
               const int32_t* gold_dev, int32_t B) {
  check(!c->dense, ZO_ERR_CONFIG, "dense_mezo has no serving-path form (runtime.py:275-279): use the materialising loop");
  check(nu >= 1, ZO_ERR_CONFIG, "nu must be >= 1");
  check(B >= 1 && B <= c->d.max_batch, ZO_ERR_DIMENSION, "batch size out of range");
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  k_set_u64<<<1, 1, 0, c->st>>>(c->d_step, step);
  ZO_CUDA_TRY(cudaMemcpyAsync(c->tok, tokens_dev, (size_t)B * c->T * 4, cudaMemcpyDeviceToDevice, c->st));
  const size_t ng = (size_t)B * c->d.opt_len * 4;
  ZO_CUDA_TRY(cudaMemcpyAsync(c->gold, gold_dev, ng, cudaMemcpyDeviceToDevice, c->st));
  ZO_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(c->gold) + ng, gold_dev, ng, cudaMemcpyDeviceToDevice, c->st));
  const int64_t wstart = lozo ? (int64_t)((step / (uint64_t)nu) * (uint64_t)nu) : (int64_t)step;
  if (!lozo || wstart != c->v_window) {
    if (lozo && c->a_dirty) fold_all(c);
    sampler_launch(c->planV, seed, c->d_step, (uint32_t)nu, c->V, c->st);
    write_vext_all(c);
    c->v_window = wstart;
  }
}

// directions (U, z), probes and paired scoring of the staged step: per-example NLLs in the ctx
void score_body(zo_ctx* c, uint64_t seed, double eps, int32_t B) {
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  sampler_launch(c->planU, seed, c->d_step, 1, c->U, c->st);
  sample_z(c, seed);
  const double scale = lozo ? 1.0 : 1.0 / std::sqrt((double)c->r);
  launch_prep_probe(lozo ? c->A : nullptr, c->U, c->su, eps, scale, c->Pp, c->Pm, c->st);
  vec_probe(c, eps);
  do_score(c, B, 2);
}

// canonical mean / c / update over B_total gathered NLLs
void apply_body(zo_ctx* c, double eps, double lr, int32_t divide_by_r, int32_t B_total) {
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  launch_coefficient(c->nll, B_total, eps, lr, lozo ? divide_by_r : 0, c->r, c->out4, c->abort_flag, c->st);
  if (lozo)
    launch_update(c->A, c->U, c->su, c->out4, c->abort_flag, c->st);
  else
    launch_dense_update_dev(c, lr, c->out4, c->abort_flag);
  vec_update(c, c->out4, lr, c->abort_flag);
}

// q-direction apply: regenerate the G counter-keyed U's (steps d_base + g) and apply the G
// gathered coefficients in g order
void qdir_apply_body(zo_ctx* c, uint64_t seed, int32_t G, double lr, const double* out4_all_dev) {
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  for (int32_t g = 0; g < G; ++g) {
    k_step_from_base<<<1, 1, 0, c->st>>>(c->d_step, c->d_base, (uint64_t)g);
    sampler_launch(c->planU, seed, c->d_step, 1, c->U, c->st);
    sample_z(c, seed);
    const double* o4 = out4_all_dev + 4 * (size_t)g;
    vec_update(c, o4, lr, nullptr);
    if (lozo) {
      launch_update(c->A, c->U, c->su, o4, nullptr, c->st);
    } else {
      // factorized: V is keyed by the step too (zo_engine.py:181-191)
      sampler_launch(c->planV, seed, c->d_step, 1, c->V, c->st);
      launch_dense_update_dev(c, lr, o4, nullptr);
    }
  }
  // the ctx out4 mirrors the last direction (zo_read_out4)
  ZO_CUDA_TRY(cudaMemcpyAsync(c->out4, out4_all_dev + 4 * (size_t)(G - 1), 32, cudaMemcpyDeviceToDevice, c->st));
}

// Launch `body` as a captured CUDA graph: the first use of a key runs it eagerly (warming
// plans / attributes) and captures it; later uses with the same key replay the graph.
template <class F>
void run_graph(zo_ctx* c, zo_ctx::GraphSlot& gs, const std::vector<uint64_t>& key, F&& body) {
  if (gs.valid && gs.key == key) {
    ZO_CUDA_TRY(cudaGraphLaunch(gs.exec, c->st));
    return;
  }
  body();
  if (!c->cap_st) ZO_CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking));
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  if (gs.exec) {
    ZO_CUDA_TRY(cudaGraphExecDestroy(gs.exec));
    gs.exec = nullptr;
  }
  gs.valid = false;
  cudaStream_t user = c->st;
  c->st = c->cap_st;
  cudaGraph_t graph = nullptr;
  try {
    ZO_CUDA_TRY(cudaStreamBeginCapture(c->cap_st, cudaStreamCaptureModeThreadLocal));
    body();
    ZO_CUDA_TRY(cudaStreamEndCapture(c->cap_st, &graph));
  } catch (...) {
    c->st = user;
    throw;
  }
  c->st = user;
  ZO_CUDA_TRY(cudaGraphInstantiate(&gs.exec, graph, 0));
  size_t n = 0;
  ZO_CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  ZO_CUDA_TRY(cudaGraphGetNodes(graph, nodes.data(), &n));
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    ZO_CUDA_TRY(cudaGraphNodeGetType(nd, &ty));
    k += ty == cudaGraphNodeTypeKernel;
  }
  gs.kernels = k;
  ZO_CUDA_TRY(cudaGraphDestroy(graph));
  gs.key = key;
  gs.valid = true;
}

uint64_t dbits(double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  return u;
}
}  // namespace

extern "C" int zo_step_score_async(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, double eps,
                                   const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B) {
  ZO_API_BEGIN
  stage_dev(c, seed, step, nu, tokens_dev, gold_dev, B);
  score_body(c, seed, eps, B);
  return ZO_OK;
  ZO_API_END
}

extern "C" int zo_step_apply_async(zo_ctx* c, double eps, double lr, int32_t divide_by_r, int32_t B_total) {
  ZO_API_BEGIN
  apply_body(c, eps, lr, divide_by_r, B_total);
  if (c->d.estimator == ZO_EST_LOZO) c->a_dirty = true;
  return ZO_OK;
  ZO_API_END
}

// The two halves of the multi-GPU exact-mode step as captured graphs (one graph launch each
// instead of ~370 kernel launches); staging and window work stay eager in front of the score
// graph, the NLL all-gather runs between the two.
extern "C" int zo_step_score_graph(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, double eps,
                                   const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B) {
  ZO_API_BEGIN
  stage_dev(c, seed, step, nu, tokens_dev, gold_dev, B);
  run_graph(c, c->gs_score, {seed, (uint64_t)B, dbits(eps)}, [&] { score_body(c, seed, eps, B); });
  return ZO_OK;
  ZO_API_END
}

extern "C" int zo_step_apply_graph(zo_ctx* c, double eps, double lr, int32_t divide_by_r, int32_t B_total) {
  ZO_API_BEGIN
  run_graph(c, c->gs_apply, {(uint64_t)B_total, dbits(eps), dbits(lr), (uint64_t)divide_by_r},
            [&] { apply_body(c, eps, lr, divide_by_r, B_total); });
  if (c->d.estimator == ZO_EST_LOZO) c->a_dirty = true;
  return ZO_OK;
  ZO_API_END
}

extern "C" int zo_step_async(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, double eps, double lr,
                             int32_t divide_by_r, const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B) {
  int rc = zo_step_score_async(c, seed, step, nu, eps, tokens_dev, gold_dev, B);
  if (rc) return rc;
  return zo_step_apply_async(c, eps, lr, divide_by_r, B);
}

// Directions (U), probes, paired scoring, coefficient and update for the step in
// d_step: the part of a step that is identical every step (graph body).
static void step_body(zo_ctx* c, uint64_t seed, double eps, double lr, int32_t divide_by_r, int32_t B) {
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  sampler_launch(c->planU, seed, c->d_step, 1, c->U, c->st);
  sample_z(c, seed);
  const double scale = lozo ? 1.0 : 1.0 / std::sqrt((double)c->r);
  launch_prep_probe(lozo ? c->A : nullptr, c->U, c->su, eps, scale, c->Pp, c->Pm, c->st);
  vec_probe(c, eps);
  do_score(c, B, 2);
  launch_coefficient(c->nll, B, eps, lr, lozo ? divide_by_r : 0, c->r, c->out4, c->abort_flag, c->st);
  if (lozo)
    launch_update(c->A, c->U, c->su, c->out4, c->abort_flag, c->st);
  else
    launch_dense_update_dev(c, lr, c->out4, c->abort_flag);
  vec_update(c, c->out4, lr, c->abort_flag);
}

// The step body as one CUDA-graph launch: captured once per (seed, B, eps, lr,
// divide_by_r) -- the first use of a key runs eagerly (warming plans / attributes),
// then captures -- and replayed afterwards.
static void graph_body(zo_ctx* c, uint64_t seed, double eps, double lr, int32_t divide_by_r, int32_t B) {
  const zo_ctx::GKey key{seed, B, divide_by_r, eps, lr};
  if (!c->gkey_valid || !(key == c->gkey)) {
    // first use of this key: run eagerly (also warms attributes/plans), then capture
    step_body(c, seed, eps, lr, divide_by_r, B);
    if (!c->cap_st) ZO_CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking));
    ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
    if (c->gexec) {
      ZO_CUDA_TRY(cudaGraphExecDestroy(c->gexec));
      c->gexec = nullptr;
    }
    cudaStream_t user = c->st;
    c->st = c->cap_st;
    cudaGraph_t graph = nullptr;
    try {
      ZO_CUDA_TRY(cudaStreamBeginCapture(c->cap_st, cudaStreamCaptureModeThreadLocal));
      step_body(c, seed, eps, lr, divide_by_r, B);
      ZO_CUDA_TRY(cudaStreamEndCapture(c->cap_st, &graph));
    } catch (...) {
      c->st = user;
      throw;
    }
    c->st = user;
    ZO_CUDA_TRY(cudaGraphInstantiate(&c->gexec, graph, 0));
    {
      // kernels per replay (the bench's gpu_launches claim counts them from here)
      size_t n = 0;
      ZO_CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &n));
      std::vector<cudaGraphNode_t> nodes(n);
      ZO_CUDA_TRY(cudaGraphGetNodes(graph, nodes.data(), &n));
      int k = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        ZO_CUDA_TRY(cudaGraphNodeGetType(nd, &ty));
        k += ty == cudaGraphNodeTypeKernel;
      }
      c->graph_kernels = k;
    }
    ZO_CUDA_TRY(cudaGraphDestroy(graph));
    c->gkey = key;
    c->gkey_valid = true;
  } else {
    ZO_CUDA_TRY(cudaGraphLaunch(c->gexec, c->st));
  }
}

// zo_step_async as one CUDA-graph launch: the ~370 kernels of the step body are
// captured once per (seed, B, eps, lr, divide_by_r) and replayed; the step index,
// token staging and window work (V resampling / fold) stay eager in front of it.
extern "C" int zo_step_graph(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, double eps, double lr,
                             int32_t divide_by_r, const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B) {
  ZO_API_BEGIN
  check(!c->dense, ZO_ERR_CONFIG, "dense_mezo has no serving-path form (runtime.py:275-279): use the materialising loop");
  check(nu >= 1, ZO_ERR_CONFIG, "nu must be >= 1");
  check(B >= 1 && B <= c->d.max_batch, ZO_ERR_DIMENSION, "batch size out of range");
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  k_set_u64<<<1, 1, 0, c->st>>>(c->d_step, step);
  ZO_CUDA_TRY(cudaMemcpyAsync(c->tok, tokens_dev, (size_t)B * c->T * 4, cudaMemcpyDeviceToDevice, c->st));
  const size_t ng = (size_t)B * c->d.opt_len * 4;
  ZO_CUDA_TRY(cudaMemcpyAsync(c->gold, gold_dev, ng, cudaMemcpyDeviceToDevice, c->st));
  ZO_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(c->gold) + ng, gold_dev, ng, cudaMemcpyDeviceToDevice, c->st));
  const int64_t wstart = lozo ? (int64_t)((step / (uint64_t)nu) * (uint64_t)nu) : (int64_t)step;
  if (!lozo || wstart != c->v_window) {
    if (lozo && c->a_dirty) fold_all(c);
    sampler_launch(c->planV, seed, c->d_step, (uint32_t)nu, c->V, c->st);
    write_vext_all(c);
    c->v_window = wstart;
  }
  graph_body(c, seed, eps, lr, divide_by_r, B);
  if (lozo) c->a_dirty = true;
  return ZO_OK;
  ZO_API_END
}

// kernels launched per zo_step_graph replay (0 before the first capture), and per
// window start in front of it (V sampler + extension columns + fold)
extern "C" int zo_graph_kernel_count(zo_ctx* c, int32_t* per_step, int32_t* per_window) {
  ZO_API_BEGIN
  *per_step = c->graph_kernels + 1;  // + the eager step-index write (k_set_u64)
  *per_window = 5 + 2 * (int32_t)c->mats.size();
  return ZO_OK;
  ZO_API_END
}

extern "C" int zo_fold_async(zo_ctx* c) {
  ZO_API_BEGIN
  if (c->d.estimator == ZO_EST_LOZO) fold_all(c);
  return ZO_OK;
  ZO_API_END
}

// ------------------------------------------------------------------ materialising-loop comparand
// baseline_loop.py:122-239 (run_baseline) on the same replica: the conventional
// training loop that writes the probe into the weights, scores each sign with its
// own forward, restores, then writes the update -- four m*n weight writes per
// matrix per step (here: three 16-bit serving-copy rewrites + one master+copy
// update in cached mode; four master+copy rewrites in recompute mode).  It is the
// cost comparand of the serving path (PAPER.md "official LoZO baseline") and keeps
// the reference's float64 arithmetic, so its parameters are bit-exact given c.
namespace {
double probe_scale(const zo_ctx* c) {
  return c->d.estimator == ZO_EST_FACTORIZED ? 1.0 / std::sqrt((double)c->r) : 1.0;
}
void baseline_pass(zo_ctx* c, int pass, double eps, bool recompute) {
  const double s = probe_scale(c);
  const double a_plus = eps * s, a_minus = (-2.0 * eps) * s;
  if (c->dense) {  // _DenseProbe on every parameter (baseline_loop.py:107-119, 172-174)
    for (auto& m : c->mats) {
      const int ldw = m.kind == K_EMBED ? (int)m.n : m.ldw, tr = m.kind == K_EMBED ? 0 : 1;
      const double* Zm = c->ZM + m.z_off;
      if (recompute)
        launch_dense_rw(2, m.W64, (int)m.m, (int)m.n, Zm, pass == 1 ? a_minus : a_plus, 0.0, nullptr, m.W16, ldw,
                        tr, c->bf16, c->st);
      else if (pass == 2)
        refresh_shadow(c, m);
      else
        launch_dense_rw(0, m.W64, (int)m.m, (int)m.n, Zm, a_plus, pass == 1 ? a_minus : 0.0, nullptr, m.W16, ldw, tr,
                        c->bf16, c->st);
    }
    if (recompute)
      launch_vec_inplace(c->VEC64, c->VZ, c->nvt, pass == 1 ? a_minus : a_plus, nullptr, c->VEC32, c->st);
    else if (pass == 2)
      launch_vec_probe(c->VEC64, c->VZ, c->nvt, 0.0, c->VEC32, c->st);
    else
      launch_vec_probe_sign(c->VEC64, c->VZ, c->nvt, eps, pass == 0 ? 1 : -1, c->VEC32, c->st);
    return;
  }
  for (auto& m : c->mats) {
    const int ldw = m.kind == K_EMBED ? (int)m.n : m.ldw, tr = m.kind == K_EMBED ? 0 : 1;
    double* Um = c->U + m.u_off;
    double* Vm = c->V + m.v_off;
    if (recompute) {  // _Probe.apply / restore(eps) arithmetic, in place (baseline_loop.py:94-104)
      const double a = pass == 1 ? a_minus : a_plus;
      launch_materialise(2, m.W64, (int)m.m, (int)m.n, Um, Vm, c->r, a, 0.0, nullptr, s, m.W16, ldw, tr, c->bf16,
                         c->st);
    } else if (pass == 2) {  // restore_matrix: the master was never modified
      refresh_shadow(c, m);
    } else {
      launch_materialise(0, m.W64, (int)m.m, (int)m.n, Um, Vm, c->r, a_plus, pass == 1 ? a_minus : 0.0, nullptr,
                         s, m.W16, ldw, tr, c->bf16, c->st);
    }
  }
  if (c->full_scope) {  // VectorProbe.set_sign(+1 / -1 / 0) (zo_engine.py:278-286)
    if (pass == 2)
      launch_vec_probe(c->VEC64, c->VZ, c->nvt, 0.0, c->VEC32, c->st);
    else
      launch_vec_probe_sign(c->VEC64, c->VZ, c->nvt, eps, pass == 0 ? 1 : -1, c->VEC32, c->st);
  }
}
void baseline_update(zo_ctx* c, double lr, bool recompute) {
  const double s = probe_scale(c);
  if (c->dense) {  // p += (-(eta*c)) z for every parameter, beta from the device coefficient
    for (auto& m : c->mats) {
      const int ldw = m.kind == K_EMBED ? (int)m.n : m.ldw, tr = m.kind == K_EMBED ? 0 : 1;
      launch_dense_rw(recompute ? 2 : 1, m.W64, (int)m.m, (int)m.n, c->ZM + m.z_off, 0.0, 0.0, c->out4, m.W16, ldw,
                      tr, c->bf16, c->st);
    }
    launch_vec_inplace(c->VEC64, c->VZ, c->nvt, 0.0, c->out4, c->VEC32, c->st);
    return;
  }
  for (auto& m : c->mats) {
    const int ldw = m.kind == K_EMBED ? (int)m.n : m.ldw, tr = m.kind == K_EMBED ? 0 : 1;
    launch_materialise(recompute ? 2 : 1, m.W64, (int)m.m, (int)m.n, c->U + m.u_off, c->V + m.v_off, c->r, 0.0,
                       0.0, c->out4, s, m.W16, ldw, tr, c->bf16, c->st);
  }
  vec_update(c, c->out4, lr, nullptr);  // VectorProbe.update with the unnormalised c
}
void baseline_directions(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu) {
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  const int64_t wstart = lozo ? (int64_t)((step / (uint64_t)nu) * (uint64_t)nu) : (int64_t)step;
  check(!c->a_dirty, ZO_ERR_CONFIG, "materialising loop on a replica with unfolded window mass");
  // the comparand writes its probes into the 16-bit serving copies (baseline_loop.py:68-119)
  check(!c->real32, ZO_ERR_CONFIG, "the materialising-loop comparand runs the 16-bit modes only");
  if (c->dense) {
    sampler_launch(c->planZM, seed, c->d_step, 1, c->ZM, c->st);
    sample_z(c, seed);
    ZO_CUDA_TRY(cudaMemsetAsync(c->Pp, 0, (size_t)c->su * 4, c->st));
    ZO_CUDA_TRY(cudaMemsetAsync(c->Pm, 0, (size_t)c->su * 4, c->st));
    return;
  }
  if (!lozo || wstart != c->v_window) {
    sampler_launch(c->planV, seed, c->d_step, (uint32_t)nu, c->V, c->st);
    write_vext_all(c);
    c->v_window = wstart;
  }
  sampler_launch(c->planU, seed, c->d_step, 1, c->U, c->st);
  sample_z(c, seed);
  // the forward reads the materialised weights: no LoRA extension (probe operands 0)
  ZO_CUDA_TRY(cudaMemsetAsync(c->Pp, 0, (size_t)c->su * 4, c->st));
  ZO_CUDA_TRY(cudaMemsetAsync(c->Pm, 0, (size_t)c->su * 4, c->st));
}
}  // namespace

// pass 0: W + eps*P (probe +1), 1: then -2eps*P (probe -1), 2: restore.  U/V of the
// step must be sampled (zo_sample_v / zo_sample_u) and the probe operands zeroed
// (zo_baseline_directions); score with zo_score(nsign = 1) between passes.
extern "C" int zo_baseline_pass(zo_ctx* c, int32_t pass, double eps, int32_t recompute) {
  ZO_API_BEGIN
  check(!c->master32, ZO_ERR_CONFIG, "the materialising loop keeps float64 masters: set update mode 0 first");
  check(pass >= 0 && pass <= 2, ZO_ERR_INPUT, "baseline pass must be 0, 1 or 2");
  baseline_pass(c, pass, eps, recompute != 0);
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

// W -= eta*c_used*P with the ctx coefficient (zo_coefficient / zo_set_coefficient)
extern "C" int zo_baseline_update(zo_ctx* c, double lr, int32_t recompute) {
  ZO_API_BEGIN
  check(!c->master32, ZO_ERR_CONFIG, "the materialising loop keeps float64 masters: set update mode 0 first");
  baseline_update(c, lr, recompute != 0);
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  return ZO_OK;
  ZO_API_END
}

// U (and V at a window start / every factorized step) for `step`, probe operands zeroed
extern "C" int zo_baseline_directions(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu) {
  ZO_API_BEGIN
  check(nu >= 1, ZO_ERR_CONFIG, "nu must be >= 1");
  set_step(c, step);
  baseline_directions(c, seed, step, nu);
  return ZO_OK;
  ZO_API_END
}

// One whole materialising-loop step, stream-ordered, device-resident inputs (bench).
extern "C" int zo_baseline_step_async(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, double eps, double lr,
                                      int32_t divide_by_r, int32_t recompute, const int32_t* tokens_dev,
                                      const int32_t* gold_dev, int32_t B) {
  ZO_API_BEGIN
  check(nu >= 1, ZO_ERR_CONFIG, "nu must be >= 1");
  check(B >= 1 && B <= c->d.max_batch, ZO_ERR_DIMENSION, "batch size out of range");
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  k_set_u64<<<1, 1, 0, c->st>>>(c->d_step, step);
  ZO_CUDA_TRY(cudaMemcpyAsync(c->tok, tokens_dev, (size_t)B * c->T * 4, cudaMemcpyDeviceToDevice, c->st));
  const size_t ng = (size_t)B * c->d.opt_len * 4;
  ZO_CUDA_TRY(cudaMemcpyAsync(c->gold, gold_dev, ng, cudaMemcpyDeviceToDevice, c->st));
  baseline_directions(c, seed, step, nu);
  baseline_pass(c, 0, eps, recompute != 0);
  do_score(c, B, 1);
  ZO_CUDA_TRY(cudaMemcpyAsync(c->nll_bl, c->nll, (size_t)B * 8, cudaMemcpyDeviceToDevice, c->st));
  baseline_pass(c, 1, eps, recompute != 0);
  do_score(c, B, 1);
  ZO_CUDA_TRY(cudaMemcpyAsync(c->nll + B, c->nll, (size_t)B * 8, cudaMemcpyDeviceToDevice, c->st));
  ZO_CUDA_TRY(cudaMemcpyAsync(c->nll, c->nll_bl, (size_t)B * 8, cudaMemcpyDeviceToDevice, c->st));
  baseline_pass(c, 2, eps, recompute != 0);
  launch_coefficient(c->nll, B, eps, lr, lozo ? divide_by_r : 0, c->r, c->out4, c->abort_flag, c->st);
  baseline_update(c, lr, recompute != 0);
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

// ------------------------------------------------------------------ q-direction mode
// SURVEY.md §8(e) mode 2: G ranks share the parameter state of macro-step t; rank
// g scores the direction, window and minibatch of reference step s = t*G + g on a
// full batch and computes its own [L+, L-, c, beta].  After the [G, 4] coefficients
// are all-gathered (32 B per rank), every rank regenerates U_s for all g from the
// counter-keyed stream and applies A += beta_g * U_g in g order (lozo), or the
// dense factorized update per g -- identical replicas, no weight traffic.
// G | nu keeps the G directions inside one window (they share V_win); G = 1 is
// exactly zo_step_async.
extern "C" int zo_qdir_score_async(zo_ctx* c, uint64_t seed, uint64_t macro_step, int32_t G, int32_t g, int32_t nu,
                                   double eps, double lr, int32_t divide_by_r, const int32_t* tokens_dev,
                                   const int32_t* gold_dev, int32_t B) {
  ZO_API_BEGIN
  check(G >= 1 && g >= 0 && g < G, ZO_ERR_CONFIG, "q-direction rank out of range");
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  check(!lozo || nu % G == 0, ZO_ERR_CONFIG, "q-direction mode needs the direction count to divide nu");
  check(!c->full_scope || G == 1, ZO_ERR_CONFIG, "q-direction mode with G > 1 supports scope lora_only only");
  stage_dev(c, seed, macro_step * (uint64_t)G + (uint64_t)g, lozo ? nu : 1, tokens_dev, gold_dev, B);
  score_body(c, seed, eps, B);
  launch_coefficient(c->nll, B, eps, lr, lozo ? divide_by_r : 0, c->r, c->out4, c->abort_flag, c->st);
  return ZO_OK;
  ZO_API_END
}

extern "C" int zo_qdir_score_graph(zo_ctx* c, uint64_t seed, uint64_t macro_step, int32_t G, int32_t g, int32_t nu,
                                   double eps, double lr, int32_t divide_by_r, const int32_t* tokens_dev,
                                   const int32_t* gold_dev, int32_t B) {
  ZO_API_BEGIN
  check(G >= 1 && g >= 0 && g < G, ZO_ERR_CONFIG, "q-direction rank out of range");
  const bool lozo = c->d.estimator == ZO_EST_LOZO;
  check(!lozo || nu % G == 0, ZO_ERR_CONFIG, "q-direction mode needs the direction count to divide nu");
  check(!c->full_scope || G == 1, ZO_ERR_CONFIG, "q-direction mode with G > 1 supports scope lora_only only");
  stage_dev(c, seed, macro_step * (uint64_t)G + (uint64_t)g, lozo ? nu : 1, tokens_dev, gold_dev, B);
  const int32_t dbr = lozo ? divide_by_r : 0;
  run_graph(c, c->gs_qscore, {seed, (uint64_t)B, dbits(eps), dbits(lr), (uint64_t)dbr}, [&] {
    score_body(c, seed, eps, B);
    launch_coefficient(c->nll, B, eps, lr, dbr, c->r, c->out4, c->abort_flag, c->st);
  });
  return ZO_OK;
  ZO_API_END
}

// The ctx's [L+, L-, c, beta] <-> an external device buffer (the all-gather's send /
// receive slots); stream-ordered.
extern "C" int zo_out4_io(zo_ctx* c, void* dev, int32_t to_ctx) {
  ZO_API_BEGIN
  check(dev != nullptr, ZO_ERR_INPUT, "null buffer");
  if (to_ctx)
    ZO_CUDA_TRY(cudaMemcpyAsync(c->out4, dev, 32, cudaMemcpyDeviceToDevice, c->st));
  else
    ZO_CUDA_TRY(cudaMemcpyAsync(dev, c->out4, 32, cudaMemcpyDeviceToDevice, c->st));
  return ZO_OK;
  ZO_API_END
}

extern "C" int zo_qdir_apply_async(zo_ctx* c, uint64_t seed, uint64_t macro_step, int32_t G, double lr,
                                   const double* out4_all_dev) {
  ZO_API_BEGIN
  check(G >= 1 && out4_all_dev != nullptr, ZO_ERR_CONFIG, "bad q-direction gather");
  k_set_u64<<<1, 1, 0, c->st>>>(c->d_base, macro_step * (uint64_t)G);
  qdir_apply_body(c, seed, G, lr, out4_all_dev);
  if (c->d.estimator == ZO_EST_LOZO) c->a_dirty = true;
  else c->v_window = -1;  // V holds the last direction's; the next score resamples it
  ZO_CUDA_TRY(cudaGetLastError());
  return ZO_OK;
  ZO_API_END
}

// zo_qdir_apply_async as a captured graph (replayed while seed, G, lr and the gather buffer
// stay the same); the macro-step base is written eagerly in front of it
extern "C" int zo_qdir_apply_graph(zo_ctx* c, uint64_t seed, uint64_t macro_step, int32_t G, double lr,
                                   const double* out4_all_dev) {
  ZO_API_BEGIN
  check(G >= 1 && out4_all_dev != nullptr, ZO_ERR_CONFIG, "bad q-direction gather");
  k_set_u64<<<1, 1, 0, c->st>>>(c->d_base, macro_step * (uint64_t)G);
  run_graph(c, c->gs_qapply, {seed, (uint64_t)G, dbits(lr), (uint64_t)(uintptr_t)out4_all_dev},
            [&] { qdir_apply_body(c, seed, G, lr, out4_all_dev); });
  if (c->d.estimator == ZO_EST_LOZO) c->a_dirty = true;
  else c->v_window = -1;
  return ZO_OK;
  ZO_API_END
}

// kernels per launch of the split-step graphs (0 before their first capture):
// [score, apply, qdir score, qdir apply]
extern "C" int zo_split_graph_kernels(zo_ctx* c, int32_t out[4]) {
  ZO_API_BEGIN
  out[0] = c->gs_score.valid ? c->gs_score.kernels : 0;
  out[1] = c->gs_apply.valid ? c->gs_apply.kernels : 0;
  out[2] = c->gs_qscore.valid ? c->gs_qscore.kernels : 0;
  out[3] = c->gs_qapply.valid ? c->gs_qapply.kernels : 0;
  return ZO_OK;
  ZO_API_END
}

extern "C" int zo_read_out4(zo_ctx* c, double* out4) {
  ZO_API_BEGIN
  ZO_CUDA_TRY(cudaMemcpyAsync(c->h_out4, c->out4, 32, cudaMemcpyDeviceToHost, c->st));
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaGetLastError());
  std::memcpy(out4, c->h_out4, 32);
  return ZO_OK;
  ZO_API_END
}

// ------------------------------------------------------------------ measurement hooks
// One eager step (zo_step_async semantics, device inputs) with a CUDA event in front of
// every kernel group of the scorer; ms[k] = device time charged to family k
// (0 embed, 1 LN, 2 qkv GEMM, 3 attention, 4 extension finalize, 5 attn_out GEMM,
// 6 ff_up GEMM, 7 ff_down GEMM, 8 last-layer tail + final LN + LM head + loss,
// 9 everything else: sampler, probes, coefficient, update), summed over the layers.
// The events between kernels cost little (PDL on/off moves the step by ~0.5%).
extern "C" int zo_profile_step(zo_ctx* c, uint64_t seed, uint64_t step, int32_t nu, double eps, double lr,
                               const int32_t* tokens_dev, const int32_t* gold_dev, int32_t B, float* ms) {
  ZO_API_BEGIN
  c->prof_on = true;
  c->prof_n = 0;
  prof_mark(c, PK_OTHER);
  int rc = zo_step_score_async(c, seed, step, nu, eps, tokens_dev, gold_dev, B);
  if (rc == ZO_OK) {
    prof_mark(c, PK_OTHER);
    rc = zo_step_apply_async(c, eps, lr, 0, B);
  }
  prof_mark(c, PK_OTHER);
  c->prof_on = false;
  if (rc != ZO_OK) return rc;
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  for (int k = 0; k < PK_N; ++k) ms[k] = 0.f;
  for (size_t i = 0; i + 1 < c->prof_n; ++i) {
    float t = 0.f;
    ZO_CUDA_TRY(cudaEventElapsedTime(&t, c->prof_ev[i], c->prof_ev[i + 1]));
    ms[c->prof_kind[i]] += t;
  }
  return ZO_OK;
  ZO_API_END
}

// Average device time (ms) of one launch of a layer-0 GEMM of the scorer at
// batch B (both signs): which = 0 qkv, 1 attn_out, 2 ff_up, 3 ff_down, 4 LM head.
// CUDA events bracket `reps` back-to-back launches on the ctx stream; the
// weights (>> L2) stream from HBM on every launch.
extern "C" int zo_bench_gemm(zo_ctx* c, int32_t which, int32_t B, int32_t reps, float* avg_ms, double* flops) {
  ZO_API_BEGIN
  check(which >= 0 && which <= 4 && reps >= 1, ZO_ERR_INPUT, "bad gemm id / reps");
  const int M = 2 * B * c->Tf;
  RowPlan& rp = row_plan(c, M);
  const GemmDesc& g = which == 0 ? rp.layers[0].qkv : which == 1 ? rp.layers[0].out
                    : which == 2 ? rp.layers[0].up : which == 3 ? rp.layers[0].down : rp.lm;
  const int l = c->d.n_layers > 1 ? 1 : 0;
  const GemmDesc& g2 = which == 0 ? rp.layers[l].qkv : which == 1 ? rp.layers[l].out
                     : which == 2 ? rp.layers[l].up : which == 3 ? rp.layers[l].down : rp.lm;
  gemm_launch(g, c->st);  // warm
  ZO_CUDA_TRY(cudaEventRecord(c->ev[0], c->st));
  // alternate two layers' weights so no launch finds its B operand in L2
  for (int i = 0; i < reps; ++i) gemm_launch((i & 1) ? g2 : g, c->st);
  ZO_CUDA_TRY(cudaEventRecord(c->ev[1], c->st));
  ZO_CUDA_TRY(cudaEventSynchronize(c->ev[1]));
  float ms = 0;
  ZO_CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  *avg_ms = ms / reps;
  const double K = (double)(g.num_kb - 1) * 64 + 16.0 * g.last_ksteps;
  *flops = 2.0 * g.M * (double)g.N * K;
  return ZO_OK;
  ZO_API_END
}

// Diagnostic timeline of one launch of a layer GEMM (which as zo_bench_gemm): per CTA 64
// globaltimer stamps (zo_gemm.h GemmDesc::trace) into host[grid * 64] and the grid size.
extern "C" int zo_trace_gemm(zo_ctx* c, int32_t which, int32_t B, uint64_t* host, int32_t cap, int32_t* grid) {
  ZO_API_BEGIN
  check(which >= 0 && which <= 4, ZO_ERR_INPUT, "bad gemm id");
  const int M = 2 * B * c->Tf;
  RowPlan& rp = row_plan(c, M);
  GemmDesc g = which == 0 ? rp.layers[0].qkv : which == 1 ? rp.layers[0].out
             : which == 2 ? rp.layers[0].up : which == 3 ? rp.layers[0].down : rp.lm;
  const int l = c->d.n_layers > 1 ? 1 : 0;
  const GemmDesc& g2 = which == 0 ? rp.layers[l].qkv : which == 1 ? rp.layers[l].out
                     : which == 2 ? rp.layers[l].up : which == 3 ? rp.layers[l].down : rp.lm;
  check(cap >= g.grid * 64, ZO_ERR_DIMENSION, "trace buffer too small");
  DevAlloc tmp;
  unsigned long long* d = tmp.get<unsigned long long>((size_t)g.grid * 64);
  for (int i = 0; i < 6; ++i) gemm_launch((i & 1) ? g2 : g, c->st);  // warm, alternating weights
  g.trace = d;
  gemm_launch(g, c->st);
  ZO_CUDA_TRY(cudaStreamSynchronize(c->st));
  ZO_CUDA_TRY(cudaMemcpy(host, d, (size_t)g.grid * 64 * 8, cudaMemcpyDeviceToHost));
  *grid = g.grid;
  return ZO_OK;
  ZO_API_END
}

// External device buffer <-> ctx per-example NLLs [2, B] (multi-GPU exact mode
// exchanges them between the scoring and the coefficient phases).
extern "C" int zo_nll_io(zo_ctx* c, void* dev, int32_t count, int32_t to_ctx) {
  ZO_API_BEGIN
  check(count >= 0 && count <= 2 * std::max(c->d.max_batch, 4096), ZO_ERR_DIMENSION, "nll count out of range");
  if (to_ctx)
    ZO_CUDA_TRY(cudaMemcpyAsync(c->nll, dev, (size_t)count * 8, cudaMemcpyDeviceToDevice, c->st));
  else
    ZO_CUDA_TRY(cudaMemcpyAsync(dev, c->nll, (size_t)count * 8, cudaMemcpyDeviceToDevice, c->st));
  return ZO_OK;
  ZO_API_END
}

// ------------------------------------------------------------------ test hooks
extern "C" int zo_test_gemm(int32_t M, int32_t N, int32_t K, int32_t lda, int32_t epi, int32_t bf16,
                            const uint16_t* A_host, const uint16_t* B_host, float* C_host) {
  ZO_API_BEGIN
  // D[M, N] = A[M, K] B[N, K]^T through the production GEMM (K2); epi in
  // {STORE16, GELU16, RESID32, STORE32}; 16-bit outputs are widened to fp32.
  check(lda >= K && lda % 8 == 0, ZO_ERR_DIMENSION, "lda must be >= K and a multiple of 8");
  int dev = 0;
  ZO_CUDA_TRY(cudaGetDevice(&dev));
  int sms = 148;
  ZO_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DevAlloc m;
  const int Mpad = (int)ceil_div(M, 128) * 128;
  uint16_t* A = m.get<uint16_t>((size_t)Mpad * lda);
  uint16_t* B = m.get<uint16_t>((size_t)N * lda);
  ZO_CUDA_TRY(cudaMemcpy(A, A_host, (size_t)M * lda * 2, cudaMemcpyHostToDevice));
  ZO_CUDA_TRY(cudaMemcpy(B, B_host, (size_t)N * lda * 2, cudaMemcpyHostToDevice));
  const bool out16 = epi == EPI_STORE16 || epi == EPI_GELU16;
  void* C = out16 ? (void*)m.get<uint16_t>((size_t)M * N) : (void*)m.get<float>((size_t)M * N);
  if (epi == EPI_RESID32) ZO_CUDA_TRY(cudaMemcpy(C, C_host, (size_t)M * N * 4, cudaMemcpyHostToDevice));
  GemmDesc g;
  gemm_plan(g, A, M, lda, B, N, lda, K, epi, bf16 != 0, C, N, sms);
  const char* e = std::getenv("ZO_STREAMK");
  if (!e || std::atoi(e) != 0)
    gemm_enable_streamk(g, m.get<float>(gemm_sk_ws_floats(sms)), m.get<unsigned>(sms + 1), sms);
  gemm_launch(g, 0);
  ZO_CUDA_TRY(cudaDeviceSynchronize());
  ZO_CUDA_TRY(cudaGetLastError());
  if (out16) {
    std::vector<uint16_t> h((size_t)M * N);
    ZO_CUDA_TRY(cudaMemcpy(h.data(), C, h.size() * 2, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < h.size(); ++i) {
      uint32_t bits;
      if (bf16) {
        bits = (uint32_t)h[i] << 16;
      } else {
        // fp16 -> fp32
        const uint32_t s = (h[i] >> 15) & 1, e = (h[i] >> 10) & 0x1f, f = h[i] & 0x3ff;
        if (e == 0) {
          float v = std::ldexp((float)f, -24);
          C_host[i] = s ? -v : v;
          continue;
        }
        bits = (s << 31) | ((e == 31 ? 255 : e - 15 + 127) << 23) | (f << 13);
      }
      std::memcpy(&C_host[i], &bits, 4);
    }
  } else {
    ZO_CUDA_TRY(cudaMemcpy(C_host, C, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  }
  return ZO_OK;
  ZO_API_END
}

// test hook of the real32 path: C[M, N] = A[M, K] . W[K, N] (W in the reference's (in, out)
// layout, float64) through the production 3xTF32 split (precise.cu) and the tf32 tcgen05
// GEMM (EPI_STORE32); A is fp32 as the scorer's activations are.
extern "C" int zo_test_gemm_tf32x3(int32_t M, int32_t N, int32_t K, const float* A_host, const double* W_host,
                                   float* C_host) {
  ZO_API_BEGIN
  check(M >= 1 && N >= 1 && K >= 1, ZO_ERR_DIMENSION, "bad GEMM shape");
  int dev = 0;
  ZO_CUDA_TRY(cudaGetDevice(&dev));
  int sms = 148;
  ZO_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DevAlloc m;
  const int Mpad = (int)ceil_div(M, 128) * 128;
  const int ldk = (int)ceil_div(3 * K, 32) * 32;
  float* A = m.get<float>((size_t)M * K);
  double* W = m.get<double>((size_t)K * N);
  float* As = m.get<float>((size_t)Mpad * ldk);
  float* Ws = m.get<float>((size_t)N * ldk);
  float* C = m.get<float>((size_t)M * N);
  ZO_CUDA_TRY(cudaMemcpy(A, A_host, (size_t)M * K * 4, cudaMemcpyHostToDevice));
  ZO_CUDA_TRY(cudaMemcpy(W, W_host, (size_t)K * N * 8, cudaMemcpyHostToDevice));
  launch_split_act(A, K, M, K, As, ldk, nullptr, nullptr, 0, M, 0, 0);
  launch_split_weight(W, K, N, nullptr, 0, Ws, ldk, 1, 0);
  GemmDesc g;
  gemm_plan(g, As, M, ldk, Ws, N, ldk, 3 * K, EPI_STORE32, 2, C, N, sms);
  gemm_launch(g, 0);
  ZO_CUDA_TRY(cudaDeviceSynchronize());
  ZO_CUDA_TRY(cudaMemcpy(C_host, C, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  return ZO_OK;
  ZO_API_END
}
