"""paper_2605_28760_b200 -- a B200-native LoZO/MeZO zeroth-order engine.

Reference-shaped API (zoserve, /root/reference/pkg/src/zoserve) over the
libzob200 C ABI (include/zob200.h): hand-written sm_100a kernels for the
direction sampler, the tcgen05 scorer, loss extraction and the low-rank
update.  No CPU fallback: every compute call goes through the CUDA library.
"""
from .errors import ConfigError, DimensionError, InputError, ScoringAbort  # noqa: F401
from .engine import ZoEngine  # noqa: F401

__version__ = "0.1.0"
