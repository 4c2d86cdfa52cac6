"""CPU checks of the product boundary: libhyt.so loads, exports every symbol that
include/hyt.h declares, fails loudly (HYT_ECUDA) without a GPU, and its host
routines (task combination, engine selection) agree with the oracle."""
import ctypes
import random

import numpy as np
import pytest

import oracle
import paper_2208_14935_b200 as hyt
from conftest import gpu_available


def test_exports_every_declared_symbol():
    declared = hyt.declared_symbols()
    assert len(declared) >= 15
    lib = ctypes.CDLL(hyt.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", hyt.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU error path")
def test_no_gpu_fails_loudly():
    with pytest.raises(hyt.HytError) as ei:
        hyt.Graph(device=0)
    assert ei.value.code == hyt.HYT_ECUDA


def test_combine_matches_oracle():
    rng = random.Random(5)
    for _ in range(2000):
        n = rng.randint(0, 50)
        p = [rng.choice([0, 1, 1, 1, 2, 3]) for _ in range(n)]
        k = rng.randint(1, 6)
        assert hyt.combine(p, k) == oracle.combine(p, k)


def test_combine_spec_examples():
    assert hyt.combine([1] * 5, 4) == [(0, 4), (4, 5)]
    assert hyt.combine([1, 2, 1], 4) == [(0, 1), (2, 3)]


def test_select_engine_matches_oracle():
    rng = random.Random(11)
    for d1 in (4, 8):
        cfg = oracle.CostCfg(d1=d1)
        for _ in range(20000):
            t = rng.choice([rng.randint(1, 20000), rng.randint(1, 9_000_000), 8192 * rng.randint(1, 8)])
            e = rng.choice([t, rng.randint(0, t), rng.randint(0, min(t, 300))])
            a = 0 if e == 0 else rng.randint(1, e)
            z = 0 if e == 0 else rng.randint(a, 2 * a + e * d1 // 128 + 1)
            assert hyt.select_engine(t, e, a, z, d1) == oracle.select(t, e, a, z, cfg), (t, e, a, z, d1)


def test_bad_arguments():
    assert hyt.hyt_combine(None, 3, 4, None) == hyt.HYT_EINVAL
    assert hyt.hyt_select_engine(None, 1, 1, 1, 1, 0) == hyt.HYT_EINVAL


def test_binding_constants_match_header():
    """The binding's flag / mode / engine constants and struct sizes follow include/hyt.h."""
    import re
    txt = open(hyt.HEADER_PATH).read()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(HYT_[A-Z_]+)\s+(-?\d+)u?", txt)}
    assert defs["HYT_NO_HUBSORT"] == hyt.HYT_NO_HUBSORT and defs["HYT_SYMMETRIC"] == hyt.HYT_SYMMETRIC
    assert defs["HYT_ADOPT_HOST"] == hyt.HYT_ADOPT_HOST
    for name, val in hyt.MODES.items():
        assert defs[f"HYT_MODE_{name.upper()}"] == val, name
    for name in ("BFS", "SSSP", "CC", "PR"):
        assert defs[f"HYT_{name}"] == getattr(hyt, f"HYT_{name}")
    # hyt_iter: 3 u64 + 6 u32 + 3 u64 + 1 double; hyt_stats ends with pull_iters, um_balloon_bytes,
    # exch_peer, host_store_bytes
    assert ctypes.sizeof(hyt.hyt_iter) == 3 * 8 + 6 * 4 + 3 * 8 + 8
    assert [f for f, _ in hyt.hyt_stats._fields_][-5:] == ["pull_iters", "um_balloon_bytes", "exch_peer",
                                                           "host_store_bytes", "record_bytes"]
    assert "uint64_t host_store_bytes;" in txt and "uint64_t record_bytes;" in txt
    assert "uint64_t pull_iters, um_balloon_bytes;" in txt and "uint32_t dir;" in txt


def test_order_units_matches_oracle():
    """A5: the scheduler's contribution-driven unit order equals oracle_order_units
    (descending unit score, ties by unit index) on random plans with many ties."""
    import oracle
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        p = rng.choice([0, 1, 1, 1, 2, 3], size=n).astype(np.uint8)
        units = hyt.combine(p, int(rng.integers(1, 6)))
        if rng.random() < 0.5:
            score = rng.integers(0, 4, size=n).astype(np.float64)          # integer hub sums: ties
        else:
            score = rng.random(n) * 10.0 ** rng.integers(-6, 3)            # delta sums
        assert hyt.order_units(units, score) == oracle.order_units(units, score)
