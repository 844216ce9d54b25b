"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports every symbol include/pscwin.h
declares, and its host-side geometry / contract logic matches the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pl():
    import paper_2407_02109_b200 as p
    return p


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "pscwin.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pscwin_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(pl):
    syms = _declared_symbols()
    assert len(syms) >= 16
    lib = pl.lib()
    for s in syms:
        assert hasattr(lib, s), f"libpscwin.so does not export {s}"
    from paper_2407_02109_b200._lib import EXPORTS
    assert sorted(EXPORTS) == syms


def test_library_is_sm100a_and_in_tree(pl):
    assert os.path.dirname(pl.LIB_PATH) == os.path.join(ROOT, "paper_2407_02109_b200")
    assert pl.lib().pscwin_version().decode().endswith("(sm_100a)")


@pytest.mark.parametrize("H,W,w,sx,sy", [(4, 4, 2, 0, 0), (4, 4, 2, 1, 1), (16, 16, 8, 4, 4), (64, 64, 16, 8, 8),
                                         (12, 20, 4, 1, 3), (7, 9, 4, 2, 1), (256, 256, 16, 8, 8)])
def test_index_map_matches_oracle(pl, H, W, w, sx, sy):
    assert pl.window_count(H, W, w, sx, sy) == oracle.window_count(H, W, w, sx, sy)
    assert np.array_equal(pl.index_map(H, W, w, sx, sy), oracle.index_map(H, W, w, sx, sy))


def test_contract_errors(pl):
    from paper_2407_02109_b200._lib import ERR_CONTRACT, PscwinError
    with pytest.raises(PscwinError) as e:
        pl.window_count(10, 12, 4)          # plain windows need divisibility
    assert e.value.status == ERR_CONTRACT
    with pytest.raises(PscwinError):
        pl.window_count(16, 16, 8, 8, 0)    # shift must be < window
    assert pl.window_count(10, 12, 4, 1, 1) == oracle.window_count(10, 12, 4, 1, 1)


def test_workspace_sizes(pl):
    import synth
    for cfg in (synth.tiny(), synth.vitb(64), synth.vitb(256, cycle_scan=1)):
        d = pl.LayerDesc.from_config(cfg)
        n = pl.workspace_bytes(d)
        T = cfg.B * cfg.H * cfg.W
        assert n >= T * cfg.C * 2 * 5  # u + qkv (3C) + O at least
    bad = pl.LayerDesc.from_config(synth.tiny(heads=3))  # C % heads != 0
    assert pl.workspace_bytes(bad) == 0


def test_null_and_alignment_checks_without_gpu(pl):
    from paper_2407_02109_b200._lib import ERR_ALIGN, ERR_CONTRACT, lib
    L = lib()
    # pad slots present but no pad row: contract error, detected before any launch
    assert L.pscwin_shifted_pad_partition(ctypes.c_void_p(16), None, 1, 4, 4, 8, 2, 1, 1, 0, ctypes.c_void_p(16),
                                          None) == ERR_CONTRACT
    assert L.pscwin_window_partition(ctypes.c_void_p(18), 1, 4, 4, 8, 2, 0, ctypes.c_void_p(16), None) == ERR_ALIGN


def test_band_plan_and_io_offsets(pl):
    # window-row bands (include/pscwin.h "row bands"): workspace planning and the exchange sizes are host logic
    import ctypes
    import synth
    from paper_2407_02109_b200._lib import BandDesc, BandIO, LayerDesc
    L = pl.lib()
    cfg = synth.vitb(256, cycle_scan=1)  # 4096^2, shifted (s = 8): 8 halo rows each way
    d = LayerDesc.from_config(cfg)
    rows = [(32 * g, 32 * g + 32) for g in range(8)]
    ios = []
    for g, (r0, r1) in enumerate(rows):
        b = BandDesc(r0, r1, g, 8)
        assert L.pscwin_band_workspace_bytes(ctypes.byref(d), ctypes.byref(b)) > 0
        io = BandIO()
        assert L.pscwin_band_io_offsets(ctypes.byref(d), ctypes.byref(b), ctypes.byref(io)) == 0
        ios.append(io)
    row = 256 * 3 * 768 * 2
    for g in range(8):
        assert ios[g].recv_prev_bytes == (8 * row if g > 0 else 0)
        assert ios[g].recv_next_bytes == (8 * row if g < 7 else 0)
        if g > 0:
            assert ios[g].send_prev_bytes == ios[g - 1].recv_next_bytes
        if g < 7:
            assert ios[g].send_next_bytes == ios[g + 1].recv_prev_bytes
        assert ios[g].hist_bytes == 3 * 1536 * 2 and ios[g].rec_bytes == 1536 * (2 + 3 * 32) * 4
    bad = [BandDesc(8, 40, 1, 8),    # not whole window rows
           BandDesc(0, 32, 1, 8),    # rank 1 cannot start at row 0
           BandDesc(224, 256, 6, 8)]  # rank 6 cannot end at H
    for b in bad:
        assert L.pscwin_band_workspace_bytes(ctypes.byref(d), ctypes.byref(b)) == 0
    # a ragged last band shorter than the halo it sends to the previous rank: H = 34, w = 8, shift 4
    # sends w - pt = 4 rows from a 2-row band; H = 36 with shift_y = 5 sends 5 rows from a 4-row band
    for H, sy, r0 in ((34, 4, 32), (36, 5, 32)):
        t = LayerDesc.from_config(synth.tiny(H=H, W=16, shift_x=4, shift_y=sy))
        io = BandIO()
        assert L.pscwin_band_io_offsets(ctypes.byref(t), ctypes.byref(BandDesc(r0, H, 2, 3)), ctypes.byref(io)) != 0
        assert L.pscwin_band_workspace_bytes(ctypes.byref(t), ctypes.byref(BandDesc(r0, H, 2, 3))) == 0
    ok = LayerDesc.from_config(synth.tiny(H=34, W=16, shift_x=4, shift_y=4))
    assert L.pscwin_band_io_offsets(ctypes.byref(ok), ctypes.byref(BandDesc(24, 34, 2, 3)), ctypes.byref(BandIO())) == 0
    col = LayerDesc.from_config(cfg.replace(scan_order=synth.SCAN_COL_MAJOR))
    assert L.pscwin_band_workspace_bytes(ctypes.byref(col), ctypes.byref(BandDesc(0, 32, 0, 8))) == 0
    # window-major: bands of whole window rows of a window-divisible grid are contiguous segments (and need the
    # permuted xz / gated-output buffers on top of the row-major plan); a ragged grid is rejected
    wm = LayerDesc.from_config(cfg.replace(scan_order=synth.SCAN_WINDOW_MAJOR))
    assert (L.pscwin_band_workspace_bytes(ctypes.byref(wm), ctypes.byref(BandDesc(32, 64, 1, 8))) >
            L.pscwin_band_workspace_bytes(ctypes.byref(d), ctypes.byref(BandDesc(32, 64, 1, 8))) > 0)
    wm_ragged = LayerDesc.from_config(synth.tiny(H=36, W=16, cycle_scan=1, scan_order=synth.SCAN_WINDOW_MAJOR))
    assert L.pscwin_band_workspace_bytes(ctypes.byref(wm_ragged), ctypes.byref(BandDesc(24, 36, 2, 3))) == 0


@pytest.mark.parametrize("scales,w,sx,sy", [([(4, 4), (2, 2)], 2, 0, 0), ([(16, 16), (8, 8), (24, 8)], 8, 4, 4),
                                            ([(12, 20), (7, 9), (3, 3), (5, 1)], 4, 1, 3)])
def test_ms_index_map_matches_oracle(pl, scales, w, sx, sy):
    desc = pl.MSDesc.make(synth.tiny(window=w, shift_x=sx, shift_y=sy), scales)
    assert np.array_equal(pl.ms_index_map(desc), oracle.ms_index_map(scales, w, sx, sy))


def test_ms_workspace_and_contract(pl):
    cfg = synth.vitb(64)
    full = pl.MSDesc.make(cfg.replace(B=2), [(64, 64), (128, 128), (256, 256)], 1, 2)
    assert pl.ms_workspace_bytes(full) > 0
    bad = pl.MSDesc.make(cfg.replace(shift_x=0, shift_y=0), [(64, 64), (40, 40)], 1, 0)  # 40 % 16 != 0 (plain)
    assert pl.ms_workspace_bytes(bad) == 0
    none = pl.MSDesc.make(cfg, [(64, 64)], 0, 0)                                          # nothing to run
    assert pl.ms_workspace_bytes(none) == 0


def test_status_strings_cover_nccl_errors():
    import paper_2407_02109_b200._lib as L
    for st in (L.ERR_NCCL, L.ERR_TIMEOUT):
        assert L.lib().pscwin_status_string(st).decode() != "unknown status"
