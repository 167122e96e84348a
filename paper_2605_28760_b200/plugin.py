"""Level-A drop-in: run the UNMODIFIED reference (zoserve) with the B200 scorer.

* ``ReferenceScorer(params, mcfg, state)`` implements zoserve's ``scorer``
  protocol (zo_engine.py:340-346) for ``zoserve.zo_engine.lozo_step(...,
  scorer=...)`` / ``estimate_coefficient``: on the +1 call it uploads the
  reference AdapterState's window slot (A, V) and probe (U) to the device,
  scores both probes in one fused launch and returns L+; the -1 call returns
  the cached L-.  Pure: it never writes the reference's params or state.
* ``install_into_zoserve(zoserve)`` patches ``zoserve.runtime.forward_score``
  (the name ``_MeteredScorer`` calls, runtime.py:28,168-177),
  ``zoserve.runtime.evaluate_split`` (runtime.py:295-301, single-token options: one
  device composition scores both options) and ``zoserve.runtime._fold_all``
  (runtime.py:242-250) so the unmodified ``run_serving_path`` scores on the GPU; folds run on the host (the
  reference's own arithmetic) and on the device replica with the same slot
  values, so both copies stay bit-identical (k_fold_shadow restates
  numerics.py:207-235 exactly).

The reference state is duck-typed: ``entries[lid].window_slot/.perturb_slot``
with ``.A, .B, .scale`` and ``perturb_sign``, ``epsilon`` (adapter.py:53-197).

scope="full": the reference's VectorProbe writes p + eps z (sign +1) and then
p - eps z (sign -1) into the 1-D params in place before each scorer call
(zo_engine.py:269-295, on_sign).  The scorer re-uploads the 1-D params whenever
they changed since the last call and then serves only the half of the fused
pair whose LN rows carry them (no L- cache across a vector change).
"""
from __future__ import annotations

import numpy as np

from .engine import A as SLOT_A, U as SLOT_U, V as SLOT_V, ZoEngine
from .errors import ConfigError
from .numerics import canonical_mean


def _engine_from_reference(params, mcfg, rank: int, batch_size: int, precision: str) -> ZoEngine:
    eng = ZoEngine(mcfg.vocab, mcfg.dim, mcfg.n_layers, mcfg.n_heads, mcfg.prompt_len, opt_len=1,
                   max_batch=max(16, batch_size), rank=rank, precision=precision)
    eng.upload(params)
    return eng


def upload_reference_slots(eng: ZoEngine, state, with_probe: bool) -> None:
    """Window A/V and probe U of a reference AdapterState -> device arenas."""
    r = eng.rank
    A = {l: np.zeros((eng.shapes[l][0], r)) for l in eng.lids}
    U = {l: np.zeros((eng.shapes[l][0], r)) for l in eng.lids}
    V = eng.split(SLOT_V, eng.get_slot(SLOT_V))
    for lid, e in state.entries.items():
        if any(s.rank for s in getattr(e, "update_slots", [])):
            raise ConfigError("frozen update slots present: fold before GPU scoring")
        B = None
        ws = e.window_slot
        if ws is not None and ws.rank:
            if ws.scale != 1.0:
                raise ConfigError("window slot scale must be 1")
            A[lid], B = ws.A, ws.B
        ps = e.perturb_slot
        if with_probe and ps is not None and ps.rank:
            if ps.scale != 1.0:
                raise ConfigError("probe scale must be 1 for the lozo device scorer")
            U[lid] = ps.A
            if B is not None and not np.array_equal(B, ps.B):
                raise ConfigError("window slot and probe must share V")
            B = ps.B
        if B is not None:
            V[lid] = B
    eng.set_slot(SLOT_V, eng.join(SLOT_V, V))
    eng.set_slot(SLOT_A, eng.join(SLOT_A, A))
    eng.set_slot(SLOT_U, eng.join(SLOT_U, U))


class ReferenceScorer:
    """zoserve ``scorer`` on the B200 engine (fused +-eps pair, cached L-)."""

    def __init__(self, params, mcfg, state, rank: int = 2, batch_size: int = 16, precision: str = "fp16",
                 engine: ZoEngine | None = None):
        self.state = state
        self.params = params
        self.eng = engine or _engine_from_reference(params, mcfg, rank, batch_size, precision)
        self._cached = None
        self._vecs = {k: np.array(v, dtype=np.float64) for k, v in params.items() if np.ndim(v) == 1}

    def _sync_vectors(self) -> bool:
        """Upload 1-D params the host changed (VectorProbe); True if any changed."""
        changed = {}
        for k, v in self.params.items():
            if np.ndim(v) == 1 and not np.array_equal(v, self._vecs.get(k)):
                changed[k] = np.array(v, dtype=np.float64)
        if changed:
            self.eng.upload(changed)
            self._vecs.update(changed)
        return bool(changed)

    def _tokens(self, batch):
        gold = batch.option_array()[batch.golds]
        return np.concatenate([batch.prompts, gold], axis=1), gold

    def _fingerprint(self):
        """Adapter version for the L- cache: which slot objects are
        installed and a checksum of their factors -- an edit between the +1 and -1
        calls (outside the reference's own estimate_coefficient) forces a re-score."""
        ids, acc = [], 0.0
        for lid in sorted(self.state.entries):
            e = self.state.entries[lid]
            for sl in (e.window_slot, e.perturb_slot):
                if sl is None:
                    ids.append(None)
                    continue
                ids.append((id(sl), id(sl.A), id(sl.B), float(sl.scale)))
                acc += float(np.sum(sl.A)) + float(np.sum(sl.B))
        return hash(tuple(ids)), acc, self.state.epsilon

    def __call__(self, batch) -> float:
        sign = self.state.perturb_sign
        key = (batch.batch_id, self._fingerprint())
        if self._sync_vectors():
            self._cached = None  # the -1 probe moved the 1-D params: score it afresh
        if sign == -1 and self._cached is not None and self._cached[0] == key:
            lm = self._cached[1]
            self._cached = None
            return lm
        tokens, gold = self._tokens(batch)
        probe = sign != 0 and any(e.perturb_slot is not None for e in self.state.entries.values())
        upload_reference_slots(self.eng, self.state, probe)
        if not probe:
            self.eng.prepare_probe(self.state.epsilon, 1)
            return canonical_mean(self.eng.score(tokens, gold, nsign=1)[0])
        self.eng.prepare_probe(self.state.epsilon, 0)
        nll = self.eng.score(tokens, np.stack([gold, gold]), nsign=2)
        lp, lm = canonical_mean(nll[0]), canonical_mean(nll[1])
        if sign == 1:
            self._cached = (key, lm)
            return lp
        return lm


def evaluate_on_engine(eng: ZoEngine, prompts, golds, options) -> tuple[float, float]:
    """``evaluate_split``'s (loss, accuracy) (model.py:444-460, 247-269) on the device for
    single-token options: the option token is causally invisible to the scored row
    (SURVEY.md §0 fact 8), so one composition scores both options at once -- gold NLL
    -> canonical mean over the whole split, argmax of -NLL_j with ties to the lowest j."""
    opts = np.asarray(options, dtype=np.int64)
    prompts = np.asarray(prompts)
    golds = np.asarray(golds, dtype=np.int64)
    nll = np.empty((len(opts), prompts.shape[0]))
    mb = eng.max_batch
    for i in range(0, prompts.shape[0], mb):
        p = prompts[i:i + mb]
        tokens = np.concatenate([p, opts[golds[i:i + mb]]], axis=1)
        for j0 in range(0, len(opts), 2):  # the two halves of one launch score two options
            js = list(range(j0, min(j0 + 2, len(opts))))
            gold = np.stack([np.tile(opts[j], (p.shape[0], 1)) for j in js])
            eng.prepare_probe(0.0, 1)
            out = eng.score(tokens, gold, nsign=len(js))
            for k, j in enumerate(js):
                nll[j, i:i + mb] = out[k]
    loss = canonical_mean(nll[golds, np.arange(prompts.shape[0])])
    picks = np.argmax(-nll.T, axis=1)  # first max wins ties (model.py:267)
    return loss, float(np.mean(picks == golds))


def install_into_zoserve(zoserve, rank: int = 2, batch_size: int = 16, precision: str = "fp16"):
    """Patch the unmodified reference so run_serving_path scores on the B200.
    Returns an ``uninstall()`` callable."""
    rt = zoserve.runtime
    orig_fs, orig_fold, orig_eval = rt.forward_score, rt._fold_all, getattr(rt, "evaluate_split", None)
    engines: dict[int, tuple[object, ReferenceScorer]] = {}

    def scorer_for(params, cfg, state):
        ent = engines.get(id(params))
        if ent is None or ent[0] is not params:
            ent = (params, ReferenceScorer(params, cfg, state, rank, batch_size, precision))
            engines[id(params)] = ent
        ent[1].state = state
        return ent[1]

    def forward_score(params, cfg, batch, view=None, precision="real64"):
        # same signature as model.py:223-229; _MeteredScorer passes view= and precision= by keyword
        if view is None:
            return orig_fs(params, cfg, batch, view=view, precision=precision)
        state = view.__closure__[0].cell_contents  # AdapterState.view() closure (adapter.py:181-190)
        return scorer_for(params, cfg, state)(batch)

    def fold_all(state, params, meter):
        ent = engines.get(id(params))
        if ent is not None:
            upload_reference_slots(ent[1].eng, state, with_probe=False)
            ent[1].eng.fold()  # device replica: same k-ascending float64 arithmetic
        return orig_fold(state, params, meter)

    def evaluate_split(params, cfg, data, split="dev", view=None, precision="real64"):
        # runtime.py:295-301 evaluates through the name it imported from model.py
        options = data.config.options
        if view is None or any(len(o) != 1 for o in options):
            return orig_eval(params, cfg, data, split, view, precision)
        state = view.__closure__[0].cell_contents
        sc = scorer_for(params, cfg, state)
        upload_reference_slots(sc.eng, state, with_probe=False)
        prompts, golds = data.splits[split]
        return evaluate_on_engine(sc.eng, prompts, golds, options)

    rt.forward_score, rt._fold_all = forward_score, fold_all
    if orig_eval is not None:
        rt.evaluate_split = evaluate_split

    def uninstall():
        rt.forward_score, rt._fold_all = orig_fs, orig_fold
        if orig_eval is not None:
            rt.evaluate_split = orig_eval

    return uninstall
