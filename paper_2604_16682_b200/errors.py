"""Exception types of the drop-in API (mirror of agentsim/errors.py:1-13).

The host mirror raises exactly the reference's exception classes so callers
written against ``agentsim`` keep working: validation problems are
``ConfigurationError`` (a ``ValueError``) raised *before* any GPU work,
malformed trace files are ``TraceFormatError``, and engine invariant
violations reported by the device status word are ``SimulationError``.
"""


class ConfigurationError(ValueError):
    """A configuration value or combination of values is invalid."""


class TraceFormatError(ValueError):
    """A trace file is malformed or violates trace invariants."""


class SimulationError(RuntimeError):
    """Engine state-machine misuse or an engine invariant violation."""
