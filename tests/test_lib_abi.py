"""CPU checks of the C-ABI library: it builds, loads without a GPU and exports every symbol that
include/*.h declares; the ctypes mirrors match the header layout; config validation (no compute)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_23278_b200 import build
    path = build.build()
    return C.CDLL(path)


def declared_functions():
    names = []
    for fn in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            names += re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\*?\s+\*?\s*(focus_[a-z_0-9]+)\s*\(", src, re.M)
    return sorted(set(names))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(lib, n), n
    from paper_2601_23278_b200.focus import EXPORTED
    assert sorted(EXPORTED) == names


def test_struct_layouts_match_header():
    from paper_2601_23278_b200.focus import focus_commit_result, focus_config, focus_req_state
    # sizes computed from include/focus.h field lists (natural alignment)
    # 22 x 4-byte fields, kv_pages, weight_seed, debug_taps, logit_scale, batch_invariant, 5 MoE fields
    assert C.sizeof(focus_config) == 22 * 4 + 8 + 8 + 3 * 4 + 5 * 4
    assert C.sizeof(focus_commit_result) == 5 * 4 + 64 * 4 * 2
    assert C.sizeof(focus_req_state) == 8 * 4 + 2 * 8 + 5 * 8 + 8 * 4 + 64 * 4 * 2


def test_config_validation(lib):
    from paper_2601_23278_b200.focus import _lib, focus_required_bytes, make_config
    from synth import get_config
    cfg = make_config(get_config("C1"))
    assert focus_required_bytes(cfg) > 0
    bad = [("alpha_num", 2), ("maxpool_kernel", 2), ("block_size", 65), ("block_size", 0), ("n_layers", 1),
           ("n_kv_heads", 3), ("head_dim", 24), ("conf_threshold", 0.0), ("conf_threshold", 1.5),
           ("logit_scale", 3.0), ("logit_scale", -2.0), ("logit_scale", 2.0 ** 20)]
    for field, val in bad:
        c = make_config(get_config("C1"))
        setattr(c, field, val)
        assert focus_required_bytes(c) == 0, field
    for ok in (0.0, 1.0, 16.0, 0.25):                   # powers of two (0 = 1)
        c = make_config(get_config("C1"))
        c.logit_scale = ok
        assert focus_required_bytes(c) > 0, ok
    h = C.c_void_p()
    c = make_config(get_config("C1")); c.alpha_num = 1
    assert _lib().focus_init(C.byref(c), None, 0, None, C.byref(h)) == 2        # FOCUS_ERR_CONFIG
    assert _lib().focus_status_str(3) == b"device invariant violated"


def test_c3_arena_fits_b200():
    from paper_2601_23278_b200.focus import focus_required_bytes, make_config
    from synth import get_config
    n = focus_required_bytes(make_config(get_config("C3")))
    assert 16e9 < n < 150e9, n          # 16.4 GB of bf16 weights + 14.5 GB KV + workspace
