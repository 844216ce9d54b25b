"""paper_2407_02109_b200 — B200-native (sm_100a) PSCWin layer of HRSAM (arXiv 2407.02109).

The compute lives in libpscwin.so (CUDA C++, C ABI in include/pscwin.h); this package is a thin ctypes
binding with the same call names. Importing it loads the library and fails loudly if it is missing.
"""
from ._lib import (LIB_PATH, LayerDesc, LayerWeights, PscwinError, ScanDesc, launch_count, lib,  # noqa: F401
                   profile_enable, profile_read)
from .api import (PSCWinLayer, PSCWinStack, Workspace, cycle_scan, forward, index_map, layer_norm, linear,  # noqa: F401
                  qkv_project, scan_workspace_bytes, shifted_pad_partition, window_attention, window_count,
                  window_merge, window_partition, workspace_bytes)

lib()  # no silent fallback: the CUDA library must be present
