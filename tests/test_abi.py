"""The C-ABI library loads and exports every symbol include/rails.h declares;
host-side argument validation works without a GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rails.h")


@pytest.fixture(scope="module")
def L():
    from paper_2510_19262_b200 import build
    build.build()
    from paper_2510_19262_b200 import rails
    return rails


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rails_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("rails_histogram", "rails_lpt_schedule", "rails_eval", "rails_pack",
              "rails_schedule_eval",
              "rails_eval_finalize", "rails_lpt_assign", "rails_rail_offsets", "rails_check",
              "rails_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(L):
    lib = L.lib()
    out = os.popen(f"nm -D --defined-only {L.LIB_PATH}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), f"{s} not exported"
        assert hasattr(lib, s)


def test_kernels_are_sm100a(L):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {L.LIB_PATH}").read()
    assert "sm_100a" in out


def test_version_and_error_string(L):
    assert L.version() == 200
    assert isinstance(L.lib().rails_last_error(), bytes)


def test_host_validation_without_gpu(L):
    lib = L.lib()
    bad = L.topo(1, 4, 4096)  # M < 2
    sh = L.shard(1, 0, 1)
    n = ctypes.c_size_t(0)
    assert lib.rails_schedule_workspace(ctypes.byref(bad), ctypes.byref(sh), ctypes.byref(n)) == L.RAILS_EINVAL
    assert b"M=1" in lib.rails_last_error()
    for tp in (L.topo(4, 0, 4096), L.topo(4, 33, 4096), L.topo(4, 4, 0), L.topo(4, 4, 1 << 32),
               L.topo(4, 4, 4096, R2=0.0), L.topo(4, 4, 4096, R2=10.0, R1=5.0)):
        assert lib.rails_schedule_workspace(ctypes.byref(tp), ctypes.byref(sh), ctypes.byref(n)) == L.RAILS_EINVAL
    good = L.topo(4, 4, 4096)
    for s in (L.shard(0, 0, 1), L.shard(1, 3, 2), L.shard(1, -1, 1), L.shard(1, 0, 0)):
        assert lib.rails_schedule_workspace(ctypes.byref(good), ctypes.byref(s), ctypes.byref(n)) == L.RAILS_EINVAL
    assert lib.rails_schedule_workspace(ctypes.byref(good), ctypes.byref(L.shard(2, 0, 4)), ctypes.byref(n)) == 0
    assert n.value > 0
    # pack rejects rows that are not a multiple of 16 before touching the device
    rc = lib.rails_pack(ctypes.byref(good), ctypes.byref(sh), 10, 2, None, None, None, 8, None,
                        None, 24, None, None, None, 0, None)
    assert rc == L.RAILS_EINVAL
    # histogram rejects k > 32
    rc = lib.rails_histogram(ctypes.byref(good), ctypes.byref(sh), 10, 33, None, None, 8, 16,
                             None, None, None, None)
    assert rc == L.RAILS_EINVAL
    assert lib.rails_lpt_assign(0, 1, None, 0, None, None, None, None, None, 0, None) == L.RAILS_EINVAL


def test_binding_refuses_cpu_tensors(L):
    import torch
    tp, sh = L.topo(2, 2, 64), L.shard(1, 0, 2)
    with pytest.raises(ValueError):
        L.lpt_schedule(tp, sh, torch.zeros((1, 2, 2, 4), dtype=torch.int64),
                       workspace=torch.zeros(1 << 16, dtype=torch.uint8))
