"""Exception hierarchy of the denoise hot path.

Mirrors the reference's error contract (``ditplan/errors.py:6-22``):
``ConfigError(message, path)`` renders as ``"{path}: {message}"`` and keeps
``.path``; config misuse is raised in Python *before* any native call.
Native failures (a negative status from the C-ABI) surface as
:class:`NativeError`, a ``RuntimeError``.
"""

from __future__ import annotations


class PlanningError(Exception):
    """Base class for all domain errors (``errors.py:6-7``)."""


class ConfigError(PlanningError):
    """Invalid configuration input; ``path`` names the offending entry
    (``errors.py:10-18``)."""

    def __init__(self, message: str, path: str | None = None):
        self.path = path
        super().__init__(f"{path}: {message}" if path else message)


class DimensionError(ConfigError):
    """A geometric dimension violates a divisibility or size constraint
    (``errors.py:21-22``)."""


class NativeError(RuntimeError):
    """A C-ABI entry point returned a negative status."""
