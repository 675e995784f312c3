"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares, argument validation fails with the reference exception
classes without touching a GPU, and the host logic (wire format, sharding,
coefficients, registry) behaves like the reference."""

import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "flashomni_b200.h"


def declared():
    return re.findall(r"^FO_API [^(]*?\b(fo_\w+)\(", HEADER.read_text(), re.M)


def test_library_exports_header():
    from paper_2509_25401_b200 import _lib

    lib = _lib.load()
    names = declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures must mirror the header"
    assert lib.fo_abi_version() == 1


def test_plan_layout_sizes():
    from paper_2509_25401_b200 import _lib

    lib = _lib.load()
    n = lib.fo_plan_workspace_bytes(24, 258)
    offs = (ctypes.c_size_t * 7)()  # fo_plan_offsets writes seven offsets
    lib.fo_plan_offsets(24, 258, offs)
    assert all(o % 16 == 0 for o in offs)
    assert list(offs) == sorted(offs) and offs[-1] < n
    # items are int2 for every (head, block)
    assert offs[2] - offs[1] >= 24 * 258 * 8


def test_validation_errors_without_gpu():
    from paper_2509_25401_b200 import _lib
    from paper_2509_25401_b200.errors import ConsistencyError, ParameterError, ShapeError

    with pytest.raises(ConsistencyError):  # pool_n < 1 (symbols.py:67-68)
        _lib.call("fo_encode_symbols", None, None, 1, 4, 4, 0, None, None, None, None)
    with pytest.raises(ParameterError):  # head_dim other than 128
        _lib.call("fo_sparse_attention", None, None, None, 256, 1, 64, None, 2, 2, 1, None, 1.0, 0,
                  None, None, None, 0, None, None, None)
    with pytest.raises(ShapeError):  # symbols dimensioned wrongly
        _lib.call("fo_sparse_attention", None, None, None, 256, 1, 128, None, 3, 3, 1, None, 1.0, 0,
                  None, None, None, 0, None, None, None)
    with pytest.raises(ShapeError):
        _lib.call("fo_gemm_q", None, 256, 100, None, 1, 128, None, None, None, 1e-6, None, 1, None,
                  None)


def test_symbol_wire_format():
    from paper_2509_25401_b200 import ConsistencyError, SymbolBuffer

    import oracle

    rng = np.random.default_rng(4)
    cb, sb = oracle.random_masks(rng, 12, 20, 2)
    ref = oracle.build_symbols(cb, sb, 2)
    buf = SymbolBuffer(s_c=ref.s_c, s_s=ref.s_s, rows=12, cols=20, pool_n=2)
    back = SymbolBuffer.from_bytes(buf.to_bytes())
    assert back == buf
    blob = bytearray(buf.to_bytes())
    blob[12] = 99  # version field
    with pytest.raises(ConsistencyError):
        SymbolBuffer.from_bytes(bytes(blob))
    with pytest.raises(ConsistencyError):
        SymbolBuffer.from_bytes(buf.to_bytes()[:-1])
    with pytest.raises(ConsistencyError):
        SymbolBuffer(s_c=b"", s_s=ref.s_s, rows=12, cols=20, pool_n=2)


def test_wire_format_matches_reference_blobs():
    from paper_2509_25401_b200 import SymbolBuffer

    g = np.load(ROOT / "tests" / "golden" / "codec.npz")
    for c in range(int(g["n_cases"])):
        blob = g[f"c{c}_blob"].tobytes()
        buf = SymbolBuffer.from_bytes(blob)
        assert buf.to_bytes() == blob
        assert buf.s_c == g[f"c{c}_sc"].tobytes()


def test_storage_bound_33k():
    # test_symbols.py:160-173: 32768 tokens, 64-token blocks, pool 2 -> < 9 KB per head
    from paper_2509_25401_b200.symbols import ceil_div

    t = ceil_div(32768, 64)
    comp = ceil_div(t, 2)
    assert comp * ceil_div(comp, 8) < 9 * 1024
    # the B200 geometry (C4): 258 blocks of 128 tokens, pool 1
    assert 258 * ceil_div(258, 8) == 8514


def test_forecast_coefficients():
    from paper_2509_25401_b200 import forecast_coefficients

    assert forecast_coefficients(2, 4, 2).tolist() == [1.0, 0.5]
    assert forecast_coefficients(1, 6, 3).dtype == np.float32


def test_shard_heads():
    from paper_2509_25401_b200 import ParameterError, shard_heads

    assert shard_heads(24, 8, 3) == [9, 10, 11]
    assert sum((shard_heads(24, 4, r) for r in range(4)), []) == list(range(24))
    with pytest.raises(ParameterError):
        shard_heads(24, 5, 0)


def test_backend_registry():
    from paper_2509_25401_b200 import available_backends, get_backend

    assert list(available_backends()) == ["b200"]
    assert get_backend().NAME == "b200"
    with pytest.raises(ImportError):
        get_backend("python")  # no CPU fallback backend


def test_no_oracle_in_product():
    """The product package never imports the oracle."""
    pkg = ROOT / "paper_2509_25401_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f


def test_building_block_entry_points_validate_without_gpu():
    """The reference building blocks' C entry points reject bad arguments with
    the reference exception classes before any launch."""
    from paper_2509_25401_b200 import _lib
    from paper_2509_25401_b200.errors import BoundsError, ParameterError, ShapeError

    with pytest.raises(ParameterError):  # null operands
        _lib.call("fo_online_softmax_update", None, None, None, None, None, 4, 4, 4, None, None,
                  None, None)
    with pytest.raises(ParameterError):  # pool < 1 (tensor.py:119-120)
        _lib.call("fo_mean_pool_blocks", 8, 4, 4, 0, 8, None)
    with pytest.raises(ShapeError):  # rope needs an even feature dim (tensor.py:91-92)
        _lib.call("fo_rope", 8, 8, 8, 4, 5, 8, None)
    with pytest.raises(ParameterError):  # tau_q outside [0, 1] (policy.py:101-102)
        _lib.call("fo_policy_select_cached", 8, 8, 1, 4, 1.5, 8, None)
    with pytest.raises(ParameterError):  # tau_kv outside [0, 1] (policy.py:136-137)
        _lib.call("fo_policy_select_skip", 8, 8, 1, 4, 4, 0, -0.5, 1, 8, None)
    with pytest.raises(ParameterError):  # forecast orders outside [1, 8]
        _lib.call("fo_forecast_entry", 8, 16, 0, 8, 8, None)
    with pytest.raises(BoundsError):  # entry outside the cache
        _lib.call("fo_cache_push_tile", 16, 16, 16, 256, 2, 128, 2, 1, 2, 0, None)
