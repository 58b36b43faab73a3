"""B200-native AFFMAE hot path: cluster attention, KNN merge, cluster index.

Layers:
  * ``libaffmae_b200.so`` -- CUDA kernels for sm_100a behind the C ABI
    declared in ``include/affmae_b200.h`` (sources in ``csrc/``).
  * :mod:`.capi`  -- ctypes binding of that ABI.
  * :mod:`.ops`   -- torch-device wrappers (device-resident step, bench).
  * :mod:`.inputs`-- synthetic workload generation (masks, coords, params).
"""
from . import capi  # noqa: F401

__version__ = "0.1.0"
