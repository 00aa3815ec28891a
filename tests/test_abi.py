"""The C-ABI library (no GPU needed): it loads, exports every function that
include/cog_b200.h declares, the ctypes binding covers each of them, and
calls that touch no device memory behave (version string, size queries,
argument validation returning COG_EINVAL before any launch)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_1705_09339_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "cog_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cog_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_entry_points():
    names = declared()
    for must in ("cog_prior_build", "cog_gmm_warmup", "cog_set_levels",
                 "cog_step", "cog_finalize", "cog_apply_pending",
                 "cog_baseline_frame", "cog_export_state",
                 "cog_import_state", "cog_step_host", "cog_version"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.build_extension()))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    assert set(declared()) <= set(_lib.EXPORTED)


def test_host_only_calls():
    lib = _lib.load()
    assert b"sm_100a" in lib.cog_version()
    assert lib.cog_accum_words(3, 2) == 7 * 3 + 2 + 6 * 3 * 2
    assert lib.cog_deepq_slots(3, 1000) == 3000
    # argument validation happens before any CUDA call
    assert lib.cog_step(None, None, None, None, None, None, None, None, 0, 0,
                        1, None) == _lib.COG_EINVAL
    g = _lib.Geom()
    g.height, g.width, g.depth, g.k, g.stride, g.streams = 4, 4, 9, 3, 2, 1
    assert lib.cog_set_levels(_lib.ref(g), None, None) == _lib.COG_EINVAL
    g.depth, g.k = 1, 12
    assert lib.cog_set_levels(_lib.ref(g), None, None) == _lib.COG_EUNSUPPORTED
    with pytest.raises(Exception):
        _lib.check(_lib.COG_EINVAL, "x")


def test_table_layout_size():
    """Tile-major hot prior (u16): per plane n_tiles x 256 bins x SL slots;
    mixture records of 16 / 32 elements (host-side arithmetic, no GPU)."""
    lib = _lib.load()
    for (h, w, st, d, floats) in [
            (480, 640, 2, 3, 3 * (640 // 16) * (480 // 2) * 256 * 32),
            (120, 160, 1, 1, 1 * (160 // 32) * 120 * 256 * 32),
            (7, 10, 3, 1, 1 * 2 * 3 * 256 * 32)]:   # cw 9: ragged edges
        g = _lib.Geom()
        g.total_pixels, g.height, g.width, g.depth = h * w, h, w, d
        g.k, g.stride, g.streams = 3, st, 1
        assert lib.cog_tabq_elems(_lib.ref(g)) == floats
    assert [lib.cog_mix_elems(k) for k in range(1, 9)] == [16] * 5 + [32] * 3
    assert lib.cog_mix_elems(0) == -1 and lib.cog_mix_elems(9) == -1
