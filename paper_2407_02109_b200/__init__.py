"""paper_2407_02109_b200 — B200-native (sm_100a) PSCWin layer of HRSAM (arXiv 2407.02109).

The compute lives in libpscwin.so (CUDA C++, C ABI in include/pscwin.h); this package is a thin ctypes
binding with the same call names. Importing it loads the library and fails loudly if it is missing.
"""
from ._lib import (CS_MULTI_SCALE, CS_NONE, CS_SINGLE_SCALE, LIB_PATH, LayerDesc, LayerWeights,  # noqa: F401
                   MSDesc, NeckDesc, PscwinError, ScanDesc, launch_count, lib, ms_index_map, profile_enable, profile_read)
from .api import (HRSAMEncoder, PSCWinLayer, PSCWinMSLayer, PSCWinStack, ms_forward, ms_workspace_bytes, neck,
                  neck_workspace_bytes, patch_embed, resize_bilinear, Workspace, cycle_scan, forward, index_map, layer_norm, linear,  # noqa: F401
                  qkv_project, scan_chunks, scan_workspace_bytes, shifted_pad_partition, window_attention, window_count,
                  window_merge, window_partition, workspace_bytes)

lib()  # no silent fallback: the CUDA library must be present
