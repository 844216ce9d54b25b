"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports every symbol include/pscwin.h
declares, and its host-side geometry / contract logic matches the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle

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
