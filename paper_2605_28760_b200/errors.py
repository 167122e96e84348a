"""Exception types, mirroring zoserve.numerics (numerics.py:40-49) and
zoserve.runtime.ScoringAbort (runtime.py:147)."""


class DimensionError(ValueError):
    """A shape or rank argument is out of its legal range."""


class ConfigError(ValueError):
    """A configuration value is malformed or inconsistent."""


class InputError(ValueError):
    """Input data violates a documented precondition."""


class ScoringAbort(RuntimeError):
    """Scoring failed (injected fault or a non-finite loss); the step is not applied."""
