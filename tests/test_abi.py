"""The C ABI library loads without a GPU and exports every entry point that
include/gdp2d.h declares; ctypes layouts match the C structs."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    text = (ROOT / "include" / "gdp2d.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gdp2d_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("gdp2d_refine", "gdp2d_collect", "gdp2d_locate", "gdp2d_claim", "gdp2d_cavity",
                 "gdp2d_flip_fixpoint", "gdp2d_predicates_batch", "gdp2d_last_error"):
        assert must in names


def test_library_exports_every_symbol(built):
    from paper_2007_00324_b200 import _abi as A
    lib = C.CDLL(str(A.LIB_DIR / "libgdp2d.so"))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_header(built):
    from paper_2007_00324_b200 import _abi as A
    assert set(declared_functions()) <= set(A.SIGNATURES)


def test_struct_layouts(built):
    from paper_2007_00324_b200 import _abi as A
    A.check_layouts()


def test_params_init_matches_reference_cos(built):
    """cos^2(theta) is computed on the host exactly as refine.hpp:195-196."""
    import math
    from paper_2007_00324_b200 import _abi as A
    p = A.Params()
    theta = math.degrees(math.asin(1 / (2 * math.sqrt(2))))
    A.engine().gdp2d_params_init(C.byref(p), theta, math.inf, 0)
    c = math.cos(theta * 3.14159265358979323846 / 180.0)
    assert p.cos2_theta == c * c
    assert p.cavity_n == 32 and p.iteration_cap == 10000 and p.split_depth_cap == 64
    assert p.rule2_filtering_enabled == 1 and p.rule4_unified_collection == 1


def test_no_device_fails_loudly(built):
    """Without a GPU the engine reports ENODEVICE instead of falling back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2007_00324_b200 import Engine
    with pytest.raises(RuntimeError, match="ENODEVICE"):
        Engine(0)
