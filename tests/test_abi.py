"""CPU-side checks of the C-ABI boundary: the shared library loads without a
GPU and exports every entry point include/hpg.h declares, and the Python
mirror binds exactly those."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hpg.h")
LIB = os.path.join(ROOT, "paper_2512_12476_b200", "libhpg.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hpg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("hpg_create", "hpg_eval", "hpg_check_memory", "hpg_balance", "hpg_search",
                 "hpg_ga_search", "hpg_sweep", "hpg_destroy"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libhpg.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.hpg_abi_version() == 3


@pytest.mark.skipif(not os.path.exists(LIB), reason="libhpg.so not built")
def test_python_binding_covers_header():
    from paper_2512_12476_b200 import hetplan
    assert sorted(hetplan.EXPORTED_SYMBOLS) == declared_functions()
    hetplan.load_library()


@pytest.mark.skipif(not os.path.exists(LIB), reason="libhpg.so not built")
def test_create_without_gpu_fails_loudly():
    """No CPU fallback: without a CUDA device hpg_create reports HPG_INTERNAL."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_12476_b200 import Engine, InternalError, load_topology, load_workflow
    wf = load_workflow(os.path.join(ROOT, "fixtures", "c1.workflow.json"))
    topo = load_topology(os.path.join(ROOT, "fixtures", "c1.topology.json"))
    with pytest.raises(InternalError):
        Engine(wf, topo)
