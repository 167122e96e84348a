"""ZoEngine -- one device-resident LoZO/MeZO model replica (one libzob200 ctx).

This is the Level-B engine behind the reference-shaped API in
``zo_engine.py`` / ``runtime.py``: parameters (float64 master + 16-bit
tensor-core shadows), the U/V/A slot arenas and all activations live in HBM;
the host only stages token ids and reads back (L+, L-, c, beta).
"""
from __future__ import annotations

import ctypes
import warnings

import numpy as np

from . import _lib
from ._lib import check, lib
from .errors import ConfigError, DimensionError

# "real32": the reference's float32 forward (model.py:149-154) as 3xTF32 tensor-core GEMMs with
# fp32 LN / attention / loss -- the parity mode.  "fp16" / "bf16": 16-bit operands, fp32
# accumulate -- the performance modes (fp16 default).
PRECISIONS = {"fp16": _lib.PREC_FP16, "bf16": _lib.PREC_BF16, "real32": _lib.PREC_FP32}
ALIASES = {"fp32": "real32"}
# "real64" (the reference's default) has no device form: float64 GEMMs are not on the tensor
# cores.  It runs the fp16 performance mode, with a warning; the float64
# parity evidence is the oracle.
REAL64_FALLBACK = "fp16"
ESTIMATORS = {"lozo_lazy": _lib.EST_LOZO, "factorized_sqrt_r": _lib.EST_FACTORIZED,
              "dense_mezo": _lib.EST_DENSE}  # dense_mezo: the materialising loop only
SCOPES = {"lora_only": _lib.SCOPE_LORA_ONLY, "full": _lib.SCOPE_FULL}
ARCHS = {"zoserve": _lib.ARCH_ZOSERVE, "opt": _lib.ARCH_OPT}


def vector_shapes(n_layers: int, dim: int, arch: str = "zoserve") -> dict[str, int]:
    """1-D params and their lengths (model.py:100-107; OPT adds the projection biases)."""
    out = {}
    for i in range(n_layers):
        for ln in ("ln1", "ln2"):
            out[f"blk{i}.{ln}.scale"] = dim
            out[f"blk{i}.{ln}.shift"] = dim
        if arch == "opt":
            out[f"blk{i}.qkv.bias"] = 3 * dim
            out[f"blk{i}.attn_out.bias"] = dim
            out[f"blk{i}.ff_up.bias"] = 4 * dim
            out[f"blk{i}.ff_down.bias"] = dim
    out["ln_f.scale"] = dim
    out["ln_f.shift"] = dim
    return out

U, V, A, Z, ZM = 0, 1, 2, 3, 4  # slot arenas (Z: 1-D directions; ZM: dense_mezo matrix directions)


def resolve_precision(precision: str) -> str:
    """Device precision for a reference precision string (model.py:149-154 accepts
    "real64" / "real32"; anything unknown is a ConfigError)."""
    if precision == "real64":
        warnings.warn("precision 'real64' has no tensor-core form: running the fp16 mode "
                      "(use 'real32' for the fp32 parity mode)", RuntimeWarning, stacklevel=3)
        return REAL64_FALLBACK
    p = ALIASES.get(precision, precision)
    if p not in PRECISIONS:
        raise ConfigError(f"unknown precision {precision!r}")
    return p


class ZoEngine:
    def __init__(self, vocab: int, dim: int, n_layers: int, n_heads: int, prompt_len: int, *,
                 opt_len: int = 1, max_batch: int = 16, rank: int = 2, estimator: str = "lozo_lazy",
                 precision: str = "fp16", device: int = 0, scope: str = "lora_only", arch: str = "zoserve",
                 max_pos: int = 2048):
        if estimator not in ESTIMATORS:
            raise ConfigError(f"estimator {estimator!r} has no device engine")
        if scope not in SCOPES:
            raise ConfigError(f"scope must be one of {tuple(SCOPES)}, got {scope!r}")
        if arch not in ARCHS:
            raise ConfigError(f"arch must be one of {tuple(ARCHS)}, got {arch!r}")
        self.scope = scope
        self.arch = arch
        self.vlens = vector_shapes(n_layers, dim, arch)
        self.precision = resolve_precision(precision)
        self.estimator = estimator
        self.rank = rank
        self.vocab, self.dim, self.n_layers, self.n_heads = vocab, dim, n_layers, n_heads
        self.prompt_len, self.opt_len, self.max_batch = prompt_len, opt_len, max_batch
        self.T = prompt_len + opt_len
        desc = _lib.ZoModelDesc(vocab, dim, n_layers, n_heads, prompt_len, opt_len, max_batch, rank,
                                ESTIMATORS[estimator], PRECISIONS[self.precision], device, SCOPES[scope],
                                ARCHS[arch], max_pos)
        h = ctypes.c_void_p()
        check(lib().zo_create(ctypes.byref(h), ctypes.byref(desc)))
        self._h = h
        n = lib().zo_num_matrices(h)
        buf = ctypes.create_string_buffer(128)
        rows, cols = ctypes.c_int64(), ctypes.c_int64()
        self.lids: list[str] = []
        self.shapes: dict[str, tuple[int, int]] = {}
        for i in range(n):
            check(lib().zo_matrix_info(h, i, buf, 128, ctypes.byref(rows), ctypes.byref(cols)))
            lid = buf.value.decode()
            self.lids.append(lid)
            self.shapes[lid] = (rows.value, cols.value)
        self.u_off, self.v_off = {}, {}
        su = sv = 0
        for lid in self.lids:
            m, nn = self.shapes[lid]
            self.u_off[lid], self.v_off[lid] = su, sv
            su += m * rank
            sv += nn * rank
        self.su, self.sv = su, sv
        self.zm_off, zm = {}, 0
        for lid in self.lids:
            self.zm_off[lid] = zm
            zm += self.shapes[lid][0] * self.shapes[lid][1]
        self.szm = zm if estimator == "dense_mezo" else 0
        self._lid_c = (ctypes.c_char_p * n)(*[l.encode() for l in self.lids])
        self.last_out4 = np.zeros(4)

    # ---------------------------------------------------------------- lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().zo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self) -> None:
        check(lib().zo_synchronize(self._h))

    def set_stream(self, stream_ptr: int) -> None:
        check(lib().zo_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    @property
    def device_bytes(self) -> int:
        b = ctypes.c_uint64()
        check(lib().zo_device_bytes(self._h, ctypes.byref(b)))
        return b.value

    # ---------------------------------------------------------------- parameters
    def init_params(self, init_seed: int, init_scale: float) -> None:
        check(lib().zo_init_params(self._h, init_seed, float(init_scale)))

    def upload(self, params) -> None:
        for lid, w in params.items():
            w = np.ascontiguousarray(w, dtype=np.float64)
            if w.ndim == 2:
                check(lib().zo_upload_matrix(self._h, lid.encode(), w.ctypes.data, w.shape[0], w.shape[1]))
            else:
                check(lib().zo_upload_vector(self._h, lid.encode(), w.ctypes.data, w.shape[0]))

    def download_vector(self, lid: str) -> np.ndarray:
        n = self.vlens.get(lid, self.dim)
        out = np.empty(n, dtype=np.float64)
        check(lib().zo_download_vector(self._h, lid.encode(), out.ctypes.data, n))
        return out

    @property
    def vids(self) -> list[str]:
        """1-D param ids in sorted order (model.py:124-125)."""
        return sorted(self.vlens)

    def update_vectors(self, lr: float) -> None:
        check(lib().zo_update_vectors(self._h, float(lr)))

    def download(self, lid: str) -> np.ndarray:
        m, n = self.shapes[lid]
        out = np.empty((m, n), dtype=np.float64)
        check(lib().zo_download_matrix(self._h, lid.encode(), out.ctypes.data, m, n))
        return out

    # ---------------------------------------------------------------- directions / slots
    def sample_u(self, seed: int, step: int) -> None:
        check(lib().zo_sample_u(self._h, seed, step))

    def sample_v(self, seed: int, step: int, nu: int) -> None:
        check(lib().zo_sample_v(self._h, seed, step, nu))

    def get_slot(self, which: int) -> np.ndarray:
        n = (self.sv if which == V else sum(self.vlens.values()) if which == Z else self.szm if which == ZM
             else self.su)
        out = np.empty(n, dtype=np.float64)
        check(lib().zo_get_slot(self._h, which, out.ctypes.data, n))
        return out

    def snapshot(self, which: int, slot: int) -> None:
        """Start an asynchronous copy of the U / V arena into host ring slot `slot` (zob200.h
        zo_slot_snapshot); read it with snapshot_wait."""
        check(lib().zo_slot_snapshot(self._h, which, slot))

    def snapshot_wait(self, which: int, slot: int) -> np.ndarray:
        """The landed snapshot (a view of engine-owned pinned memory, valid until the slot is
        reused)."""
        p = ctypes.c_void_p()
        check(lib().zo_slot_snapshot_wait(self._h, which, slot, ctypes.byref(p)))
        n = self.sv if which == V else self.su
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(n,))

    def set_slot(self, which: int, arena: np.ndarray) -> None:
        a = np.ascontiguousarray(arena, dtype=np.float64).reshape(-1)
        n = self.sv if which == V else self.su
        if a.size != n:
            raise DimensionError(f"slot arena has {a.size} values, expected {n}")
        check(lib().zo_set_slot(self._h, which, a.ctypes.data, n))

    def set_window(self, window_start: int) -> None:
        """Declare the window start whose V the arena holds (zob200.h zo_set_window)."""
        check(lib().zo_set_window(self._h, int(window_start)))

    def split(self, which: int, arena: np.ndarray) -> dict[str, np.ndarray]:
        out = {}
        for lid in self.lids:
            m, n = self.shapes[lid]
            rows = n if which == V else m
            off = (self.v_off if which == V else self.u_off)[lid]
            out[lid] = arena[off: off + rows * self.rank].reshape(rows, self.rank)
        return out

    def join(self, which: int, mats: dict) -> np.ndarray:
        return np.concatenate([np.ascontiguousarray(mats[l], dtype=np.float64).reshape(-1) for l in self.lids])

    def digest(self, which: int, arena: np.ndarray | None = None, z_arena: np.ndarray | None = None) -> int:
        """Chained FNV over (lid, factor) in sorted id order (zo_engine.py:220-261); for the
        U digest of a full-scope engine the 1-D directions (``z_arena``, default: the
        current Z slot) chain after the matrices."""
        if self.estimator == "dense_mezo":
            if which == V:
                return 0xCBF29CE484222325  # no V part: the empty chain (zo_engine.py:235-246)
            which = ZM
        if arena is None:
            arena = self.get_slot(which)
        arena = np.ascontiguousarray(arena, dtype=np.float64)
        if which == ZM:
            offs = self.zm_off
            rows = [self.shapes[l][0] * self.shapes[l][1] for l in self.lids]
        else:
            offs = self.v_off if which == V else self.u_off
            rows = [(self.shapes[l][1] if which == V else self.shapes[l][0]) * self.rank for l in self.lids]
        off_c = (ctypes.c_int64 * len(self.lids))(*[offs[l] for l in self.lids])
        cnt_c = (ctypes.c_int64 * len(self.lids))(*rows)
        h = int(lib().zo_digest_chain(self._lid_c, arena.ctypes.data, off_c, cnt_c, len(self.lids),
                                      0xCBF29CE484222325))
        if which in (U, ZM) and (self.scope == "full" or self.estimator == "dense_mezo"):
            # full scope: the dense 1-D directions chain after the matrices (zo_engine.py:256-260)
            z = np.ascontiguousarray(self.get_slot(Z) if z_arena is None else z_arena)
            vids = self.vids
            names = (ctypes.c_char_p * len(vids))(*[v.encode() for v in vids])
            lens = [self.vlens[v] for v in vids]
            zo = (ctypes.c_int64 * len(vids))(*[sum(lens[:i]) for i in range(len(vids))])
            zc = (ctypes.c_int64 * len(vids))(*lens)
            h = int(lib().zo_digest_chain(names, z.ctypes.data, zo, zc, len(vids), h))
        return h

    def sampler_flags(self) -> tuple[int, int, int]:
        f = (ctypes.c_uint32 * 3)()
        check(lib().zo_sampler_flags(self._h, f))
        return int(f[0]), int(f[1]), int(f[2])

    # ---------------------------------------------------------------- scoring / update
    def _tokens(self, tokens, gold, nsign_gold):
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        if tok.ndim != 2 or tok.shape[1] != self.T:
            raise DimensionError(f"tokens must be [B, {self.T}], got {tok.shape}")
        g = np.ascontiguousarray(gold, dtype=np.int32).reshape(nsign_gold, tok.shape[0], self.opt_len)
        return tok, g

    def prepare_probe(self, epsilon: float, sign_mode: int = 0) -> None:
        check(lib().zo_prepare_probe(self._h, float(epsilon), sign_mode))

    def score(self, tokens, gold, nsign: int = 2) -> np.ndarray:
        tok, g = self._tokens(tokens, gold, nsign)
        B = tok.shape[0]
        out = np.empty(nsign * B, dtype=np.float64)
        check(lib().zo_score(self._h, tok.ctypes.data, g.ctypes.data, B, nsign, out.ctypes.data))
        return out.reshape(nsign, B)

    def score_options(self, tokens, options) -> np.ndarray:
        """NLL of every single-token option [n_opt, B] from one sign-0 forward (zob200.h
        zo_score_options; the caller has prepared the sign-0 probe)."""
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        if tok.ndim != 2 or tok.shape[1] != self.T:
            raise DimensionError(f"tokens must be [B, {self.T}], got {tok.shape}")
        opts = np.ascontiguousarray(options, dtype=np.int32).reshape(-1)
        out = np.empty((opts.size, tok.shape[0]), dtype=np.float64)
        check(lib().zo_score_options(self._h, tok.ctypes.data, opts.ctypes.data, opts.size, tok.shape[0],
                                     out.ctypes.data))
        return out

    def coefficient(self, B: int, epsilon: float, lr: float, divide_by_r: bool) -> np.ndarray:
        out = np.empty(4)
        check(lib().zo_coefficient(self._h, B, float(epsilon), float(lr), int(divide_by_r), out.ctypes.data))
        return out

    def set_coefficient(self, out4) -> None:
        o = np.ascontiguousarray(out4, dtype=np.float64)
        check(lib().zo_set_coefficient(self._h, o.ctypes.data))

    def update_u(self) -> None:
        check(lib().zo_update_u(self._h))

    def fold(self) -> None:
        check(lib().zo_fold(self._h))

    def set_update_mode(self, mode: str) -> None:
        """Factorized dense update: "exact" (float64, bit-exact, default) or "tensor"
        (tcgen05 U V^T fused into the master/shadow update, HBM-bound; zob200.h)."""
        if mode not in ("exact", "tensor"):
            raise ConfigError(f"update mode must be 'exact' or 'tensor', got {mode!r}")
        check(lib().zo_set_update_mode(self._h, 0 if mode == "exact" else 1))
        self.update_mode = mode

    def set_schedule(self, schedule: str) -> None:
        """GEMM schedule: "fast" (stream-K tail where it pays, default) or "row_invariant"
        (no stream-K: per-example NLLs bitwise independent of the batch slicing over
        GPUs; zob200.h zo_set_schedule)."""
        if schedule not in ("fast", "row_invariant"):
            raise ConfigError(f"schedule must be 'fast' or 'row_invariant', got {schedule!r}")
        check(lib().zo_set_schedule(self._h, 0 if schedule == "fast" else 1))
        self.schedule = schedule

    def update_dense(self, lr: float) -> None:
        check(lib().zo_update_dense(self._h, float(lr)))

    def step(self, seed: int, step: int, nu: int, epsilon: float, lr: float, divide_by_r: bool,
             tokens, gold) -> np.ndarray:
        tok, g = self._tokens(tokens, gold, 1)
        out = self.last_out4
        check(lib().zo_step(self._h, seed, step, nu, float(epsilon), float(lr), int(divide_by_r),
                            tok.ctypes.data, g.ctypes.data, tok.shape[0], out.ctypes.data))
        return out.copy()

    def step_async(self, seed: int, step: int, nu: int, epsilon: float, lr: float, divide_by_r: bool,
                   tokens_dev: int, gold_dev: int, B: int) -> None:
        check(lib().zo_step_async(self._h, seed, step, nu, float(epsilon), float(lr), int(divide_by_r),
                                  ctypes.c_void_p(tokens_dev), ctypes.c_void_p(gold_dev), B))

    def step_graph(self, seed: int, step: int, nu: int, epsilon: float, lr: float, divide_by_r: bool,
                   tokens_dev: int, gold_dev: int, B: int) -> None:
        check(lib().zo_step_graph(self._h, seed, step, nu, float(epsilon), float(lr), int(divide_by_r),
                                  ctypes.c_void_p(tokens_dev), ctypes.c_void_p(gold_dev), B))

    def step_score_async(self, seed: int, step: int, nu: int, epsilon: float, tokens_dev: int, gold_dev: int,
                         B: int) -> None:
        check(lib().zo_step_score_async(self._h, seed, step, nu, float(epsilon), ctypes.c_void_p(tokens_dev),
                                        ctypes.c_void_p(gold_dev), B))

    def step_apply_async(self, epsilon: float, lr: float, divide_by_r: bool, B_total: int) -> None:
        check(lib().zo_step_apply_async(self._h, float(epsilon), float(lr), int(divide_by_r), B_total))

    def step_score_graph(self, seed: int, step: int, nu: int, epsilon: float, tokens_dev: int, gold_dev: int,
                         B: int) -> None:
        """step_score_async with the body replayed as a captured CUDA graph (zob200.h)."""
        check(lib().zo_step_score_graph(self._h, seed, step, nu, float(epsilon), ctypes.c_void_p(tokens_dev),
                                        ctypes.c_void_p(gold_dev), B))

    def step_apply_graph(self, epsilon: float, lr: float, divide_by_r: bool, B_total: int) -> None:
        check(lib().zo_step_apply_graph(self._h, float(epsilon), float(lr), int(divide_by_r), B_total))

    def qdir_score_async(self, seed: int, macro_step: int, G: int, g: int, nu: int, epsilon: float, lr: float,
                         divide_by_r: bool, tokens_dev: int, gold_dev: int, B: int) -> None:
        """q-direction mode: score reference step macro_step*G + g (zob200.h)."""
        check(lib().zo_qdir_score_async(self._h, seed, macro_step, G, g, nu, float(epsilon), float(lr),
                                        int(divide_by_r), ctypes.c_void_p(tokens_dev), ctypes.c_void_p(gold_dev),
                                        B))

    def out4_io(self, dev_ptr: int, to_ctx: bool) -> None:
        check(lib().zo_out4_io(self._h, ctypes.c_void_p(dev_ptr), int(to_ctx)))

    def qdir_apply_async(self, seed: int, macro_step: int, G: int, lr: float, out4_all_dev: int) -> None:
        check(lib().zo_qdir_apply_async(self._h, seed, macro_step, G, float(lr), ctypes.c_void_p(out4_all_dev)))

    def qdir_score_graph(self, seed: int, macro_step: int, G: int, g: int, nu: int, epsilon: float, lr: float,
                         divide_by_r: bool, tokens_dev: int, gold_dev: int, B: int) -> None:
        check(lib().zo_qdir_score_graph(self._h, seed, macro_step, G, g, nu, float(epsilon), float(lr),
                                        int(divide_by_r), ctypes.c_void_p(tokens_dev), ctypes.c_void_p(gold_dev),
                                        B))

    def qdir_apply_graph(self, seed: int, macro_step: int, G: int, lr: float, out4_all_dev: int) -> None:
        check(lib().zo_qdir_apply_graph(self._h, seed, macro_step, G, float(lr), ctypes.c_void_p(out4_all_dev)))

    def split_graph_kernels(self) -> list[int]:
        """Kernels per launch of the [score, apply, qdir score, qdir apply] graphs."""
        out = (ctypes.c_int32 * 4)()
        check(lib().zo_split_graph_kernels(self._h, out))
        return list(out)

    def fold_async(self) -> None:
        check(lib().zo_fold_async(self._h))

    def graph_kernel_count(self) -> tuple[int, int]:
        """(kernels per step_graph replay, kernels per window start)."""
        a, b = ctypes.c_int32(), ctypes.c_int32()
        check(lib().zo_graph_kernel_count(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def read_out4(self) -> np.ndarray:
        out = np.empty(4)
        check(lib().zo_read_out4(self._h, out.ctypes.data))
        return out

    def bench_gemm(self, which: int, B: int, reps: int = 20) -> tuple[float, float]:
        ms, fl = ctypes.c_float(), ctypes.c_double()
        check(lib().zo_bench_gemm(self._h, which, B, reps, ctypes.byref(ms), ctypes.byref(fl)))
        return float(ms.value), float(fl.value)

    def trace_gemm(self, which: int, B: int) -> np.ndarray:
        """Per-CTA timeline of one launch of layer GEMM `which` (zob200.h zo_trace_gemm):
        [grid, 64] globaltimer ns -- start, end, MMA and epilogue windows per tile segment."""
        buf = np.zeros(256 * 64, dtype=np.uint64)
        g = ctypes.c_int32()
        check(lib().zo_trace_gemm(self._h, which, B, buf.ctypes.data, buf.size, ctypes.byref(g)))
        return buf[: g.value * 64].reshape(g.value, 64)

    PROFILE_FAMILIES = ("embed", "ln", "qkv", "attention", "ext_finalize", "attn_out", "ff_up", "ff_down", "tail",
                        "other")

    def profile_step(self, seed: int, step: int, nu: int, epsilon: float, lr: float, tokens_dev: int,
                     gold_dev: int, B: int) -> dict:
        """Device ms per kernel family of one eager step (zob200.h zo_profile_step)."""
        f = (ctypes.c_float * 10)()
        check(lib().zo_profile_step(self._h, seed, step, nu, float(epsilon), float(lr), ctypes.c_void_p(tokens_dev),
                                    ctypes.c_void_p(gold_dev), B, f))
        return {k: float(f[i]) for i, k in enumerate(self.PROFILE_FAMILIES)}

    def nll_io(self, dev_ptr: int, count: int, to_ctx: bool) -> None:
        check(lib().zo_nll_io(self._h, ctypes.c_void_p(dev_ptr), count, int(to_ctx)))

    # ---------------------------------------------------------------- materialising-loop comparand
    def baseline_directions(self, seed: int, step: int, nu: int) -> None:
        check(lib().zo_baseline_directions(self._h, seed, step, nu))

    def baseline_pass(self, which: int, epsilon: float, recompute: bool) -> None:
        check(lib().zo_baseline_pass(self._h, which, float(epsilon), int(recompute)))

    def baseline_update(self, lr: float, recompute: bool) -> None:
        check(lib().zo_baseline_update(self._h, float(lr), int(recompute)))

    def baseline_step_async(self, seed: int, step: int, nu: int, epsilon: float, lr: float, divide_by_r: bool,
                            recompute: bool, tokens_dev: int, gold_dev: int, B: int) -> None:
        check(lib().zo_baseline_step_async(self._h, seed, step, nu, float(epsilon), float(lr), int(divide_by_r),
                                           int(recompute), ctypes.c_void_p(tokens_dev), ctypes.c_void_p(gold_dev),
                                           B))

    def last_step_ms(self) -> tuple[float, float, float]:
        f = (ctypes.c_float * 3)()
        check(lib().zo_last_step_ms(self._h, f))
        return float(f[0]), float(f[1]), float(f[2])


def test_gemm_tf32x3(A: np.ndarray, W: np.ndarray) -> np.ndarray:
    """C = A . W through the real32 path's 3xTF32 split + tf32 tcgen05 GEMM (A fp32 [M, K],
    W float64 [K, N] in the reference's (in, out) layout); returns fp32 [M, N]."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    W = np.ascontiguousarray(W, dtype=np.float64)
    M, K = A.shape
    N = W.shape[1]
    out = np.zeros((M, N), dtype=np.float32)
    check(lib().zo_test_gemm_tf32x3(M, N, K, A.ctypes.data, W.ctypes.data, out.ctypes.data))
    return out


def test_gemm(A: np.ndarray, B: np.ndarray, epi: int = 3, bf16: bool = False, C: np.ndarray | None = None,
              lda: int | None = None) -> np.ndarray:
    """Run the production tcgen05 GEMM on host arrays (A [M,K], B [N,K] as
    float16/bfloat16 bit patterns in uint16); returns fp32 [M, N]."""
    M, K = A.shape
    N = B.shape[0]
    lda = lda or ((K + 7) // 8) * 8
    Ap = np.zeros((M, lda), dtype=np.uint16)
    Ap[:, :K] = A
    Bp = np.zeros((N, lda), dtype=np.uint16)
    Bp[:, :K] = B
    out = np.zeros((M, N), dtype=np.float32) if C is None else np.ascontiguousarray(C, dtype=np.float32).copy()
    check(lib().zo_test_gemm(M, N, K, lda, epi, int(bf16), Ap.ctypes.data, Bp.ctypes.data, out.ctypes.data))
    return out
