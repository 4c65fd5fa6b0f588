"""The C-ABI library loads and exports every symbol include/tuckerplan_b200.h declares; device entry points fail
loudly (Errc.cuda) instead of falling back when there is no GPU."""
import pytest

from paper_1707_05594_b200 import Errc, TuckerplanError
from paper_1707_05594_b200._lib import LIB_PATH, exported_symbols_from_header, lib


def test_every_declared_symbol_is_exported():
    names = exported_symbols_from_header()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.tp_version().decode().startswith("tuckerplan_b200")


def test_library_is_in_tree():
    assert "paper_1707_05594_b200/lib/libtuckerplan_b200.so" in LIB_PATH.replace("\\", "/")


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1707_05594_b200 import engine
    with pytest.raises(TuckerplanError) as e:
        engine.Context(0)
    assert e.value.code == Errc.cuda
