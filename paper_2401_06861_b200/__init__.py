"""B200-native SV/DM simulation core with the reference engine's interfaces.

* ``abi``  -- ctypes binding of the C ABI (include/naqs_b200.h), used by the
  parity tests and the benchmark.
* ``naqs`` -- the reference's Python surface (``naqs._core``: Circuit,
  run_statevector, sample, expectation, run_density, density_expectation,
  DeviceNoiseModel, load_calibration, NaqsError) over the same library.

Both load the in-tree ``libnaqs_b200.so``; there is no CPU fallback.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
