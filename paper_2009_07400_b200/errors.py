"""Exception contract of the reference (errors.py:4-13, core.py:26-27).

The CUDA library reports failures through a device status word; the host
maps its codes onto these classes (see ``_native.raise_for_status``).
"""


class ConfigError(ValueError):
    """A configuration value violates an invariant (core.py:26-27)."""


class ProtocolError(RuntimeError):
    """A halo/decomposition invariant broke: atom beyond the ghost shell,
    ownership lost after exchange, plan/store mismatch (errors.py:4-5)."""


class SingularityError(ArithmeticError):
    """Two interacting atoms coincide within the cutoff (errors.py:8-9)."""


class GuardViolation(RuntimeError):
    """Atoms drifted >= verlet_buffer / 2 since the last rebuild (errors.py:12-13)."""


class NativeError(RuntimeError):
    """CUDA / NCCL failure inside the native library (status code 5)."""
