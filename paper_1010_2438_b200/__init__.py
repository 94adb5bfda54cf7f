"""B200-native bulk Gillespie direct-method simulation of CWC models with
on-line trajectory statistics (arXiv:1010.2438 hot path).

The compute lives in libcwcsim.so (include/cwc.h, csrc/); `cwc` is the thin
ctypes binding.  No oracle code is imported here.
"""
from . import cwc  # noqa: F401
from .cwc import (  # noqa: F401
    CWC_PATH_AUTO,
    CWC_PATH_THREAD,
    CWC_PATH_WARP,
    CwcError,
    Model,
    cwc_model_create,
    cwc_philox_blocks,
    cwc_simulate,
    cwc_simulate_host,
    cwc_simulate_workspace_size,
    cwc_stats_finalize,
    simulate,
)
