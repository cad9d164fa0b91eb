"""B200-native GeoDock-MA pose-search hot path (arXiv 1901.06363).

The product is the native library ``libgeodock_b200.so`` (sm_100a kernels +
C++ host runtime) behind the C-ABI in ``include/geodock_b200.h`` and the C++
drop-in header ``include/geodock_b200/geodock.hpp``.  This package holds
that library's sources (``csrc/``), its build (``build.py``), the ctypes
binding used by the tests and the benchmark (``native.py``), and the
BASELINE workload definitions (``workloads.py``).
"""
from .native import (  # noqa: F401
    Docker,
    DockResult,
    Profiles,
    GeoDockError,
    Knobs,
    LigandBatch,
    MultiDocker,
    optimal_tile_size,
    orientations,
    synth_ligands,
    synth_pocket,
)
