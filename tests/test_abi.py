"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a GPU,
exports every entry point include/adakv_b200.h declares, and its host-side
validation raises the reference's exception types before anything is launched."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "adakv_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:adakv_status|const char\*|int|int64_t)\s+(adakv_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("adakv_compress", "adakv_window_scores", "adakv_segmented_select", "adakv_gather",
                 "adakv_decode", "adakv_append_kv", "adakv_apportion", "adakv_uniform_allocation",
                 "adakv_safeguard_blend", "adakv_repair_zero_budgets", "adakv_pyramid_layer_budgets",
                 "adakv_last_error", "adakv_workspace_status", "adakv_validate_finite",
                 "adakv_clear_workspace_status", "adakv_append_rows"):
        assert must in syms


def test_library_loads_and_exports_every_symbol():
    from paper_2407_11550_b200 import _lib
    L = _lib.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert L.adakv_abi_version() == 2


def test_host_validation_mirrors_reference_throws():
    from paper_2407_11550_b200 import _lib
    L = _lib.lib()
    shape = _lib.LayerShape(1, 32, 8, 32, 4064, 128)
    cfg = _lib.PolicyConfig(2, 1, 32, 4, 0.2, 4, 4)  # even pool kernel: policies.hpp:67-68
    n = C.c_size_t()
    assert L.adakv_compress_workspace(2, C.byref(shape), C.byref(cfg), C.byref(n)) == 1
    assert b"pool_kernel must be odd" in L.adakv_last_error()
    cfg = _lib.PolicyConfig(2, 1, 32, 7, 1.5, 4, 4)  # alpha outside [0,1]: policies.hpp:69-70
    assert L.adakv_compress_workspace(2, C.byref(shape), C.byref(cfg), C.byref(n)) == 1
    assert b"alpha" in L.adakv_last_error()
    cfg = _lib.PolicyConfig(2, 1, 32, 7, 0.2, 4, 4)
    bad = _lib.LayerShape(1, 30, 8, 32, 4064, 128)  # h % g: policies.hpp:216
    assert L.adakv_compress_workspace(2, C.byref(bad), C.byref(cfg), C.byref(n)) == 1
    assert L.adakv_compress_workspace(2, C.byref(shape), C.byref(cfg), C.byref(n)) == 0
    assert n.value > 0
    # floor: layer_budget >= m*G + G (policies.hpp:229-230) -- rejected before any launch
    st = L.adakv_compress(2, C.byref(shape), C.byref(cfg), 32 * 8 + 7, None, None, None, None, 0,
                          C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), None, C.c_void_p(1),
                          None, None, None, 0, None)
    assert st == 1 and b"window-plus-one floor" in L.adakv_last_error()
    # budget helpers: reference throw sites (budget.hpp:104, 148-152, 172-174)
    assert L.adakv_uniform_allocation(3, 0, None, None) == 1
    assert L.adakv_safeguard_blend(None, 10, 10, 2, 1.5, None, None) == 1
    assert L.adakv_pyramid_layer_budgets(100, 0, 1.5, 0.5, None) == 1
    assert L.adakv_pyramid_layer_budgets(100, 3, 0.5, 1.5, None) == 1


def test_python_ops_refuse_cpu_tensors():
    torch = pytest.importorskip("torch")
    import paper_2407_11550_b200 as A
    q = torch.zeros(1, 4, 2, 8)
    k = torch.zeros(1, 2, 10, 8)
    with pytest.raises(A.InvalidArgument):
        A.compress(q, k, k, 8)


def test_host_v_must_be_pinned_cpu_tensor():
    """ops.compress accepts a host V only as a pinned, contiguous CPU tensor; anything else
    raises the reference's invalid_argument type before the library is called."""
    import torch
    from paper_2407_11550_b200 import InvalidArgument, ops
    with pytest.raises(InvalidArgument):
        ops.host_device_pointer(torch.zeros(4, 4))  # not pinned (no CUDA here: cannot pin)


def test_decode_and_append_refuse_missing_capacity_tables():
    """The capacity table is part of the boundary: decode and append reject a NULL seg_cap
    before launching (no unchecked writes past a segment, attention.hpp:126-134)."""
    from paper_2407_11550_b200 import _lib
    L = _lib.lib()
    one = C.c_void_p(16)
    st = L.adakv_decode(2, 1, 32, 8, 128, 1, one, one, one, 100, one, None, one, 64, None, None, one, one, 1 << 20,
                        0, None)
    assert st == 1 and b"segment table" in L.adakv_last_error()
    st = L.adakv_decode(2, 1, 32, 8, 128, 1, one, one, one, 100, one, one, one, 64, None, None, one, one, 1 << 20,
                        7, None)
    assert st == 1 and b"flags" in L.adakv_last_error()
    st = L.adakv_append_rows(2, 8, 1, 128, one, one, one, None, one, one, one, one, None)
    assert st == 1 and b"segment table" in L.adakv_last_error()
    assert L.adakv_validate_finite(2, one, -1, one, None) == 1
