"""The C-ABI library: loads without a GPU and exports every symbol the
header declares; the oracle libraries build and load."""
import ctypes

import pytest

import paper_2205_02473_b200._native as N


def test_every_declared_symbol_is_exported():
    assert N.check_symbols() == []


def test_abi_version():
    assert N.lib.dpro_cuda_abi_version() == 1


def test_library_is_the_in_tree_build():
    assert N.LIB_PATH.parent.name == "paper_2205_02473_b200"
    assert N.LIB_PATH.exists()


def test_create_without_gpu_returns_null():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert not N.lib.dpro_cuda_create(0)


def test_product_package_never_imports_oracle():
    import pathlib
    pkg = pathlib.Path(N.__file__).parent
    for f in pkg.rglob("*.py"):
        assert "oracle" not in f.read_text().replace("# oracle", ""), f


def test_options_rejected_without_context():
    assert N.lib.dpro_cuda_set_option(None, b"fast", 1) == N.DPRO_EINVAL
