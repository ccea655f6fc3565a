"""The C-ABI library loads on a CPU host, exports every symbol include/mbs.h declares,
and its host-only entry points (plan, factors, host gather) match the reference fixtures."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2110_12484_b200 as mbs
from paper_2110_12484_b200 import _native as N
from tests.golden_io import load_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "mbs.h")).read()
    return sorted(set(re.findall(r"\b(mbs_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(N.EXPORTS)
    assert lib.mbs_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_plan_split_native_matches_reference_fixtures():
    g = load_json("plans.json")
    for c in g["plans"]:
        p = mbs.plan_split(c["n_b"], c["n_mu_in"])
        assert p.n_mu == c["n_mu"] and p.n_s_mu == c["n_s_mu"]
        if c["sizes"] is not None:
            assert list(p.sizes) == c["sizes"]
            for mode, hexes in c["factors_hex"].items():
                assert [mbs.normalization_factor(p, k, mode).hex() for k in range(p.n_s_mu)] == hexes
                code = N.NORM_MODES[mode]
                for k in range(p.n_s_mu):
                    out = ctypes.c_double()
                    N.check(N.lib().mbs_normalization_factor(c["n_b"], c["n_mu_in"], k, code, ctypes.byref(out)))
                    assert out.value.hex() == hexes[k]
        assert list(p.index_ranges[-1]) == c["ranges_last"]
        assert sum(p.sizes) == p.n_b
    for n_b, n_mu, err in g["errors"]:
        with pytest.raises(ValueError):
            mbs.plan_split(n_b, n_mu)


def test_normalization_errors():
    p = mbs.plan_split(10, 4)
    with pytest.raises(ValueError):
        mbs.normalization_factor(p, 3, "paper_faithful")
    with pytest.raises(ValueError):
        mbs.normalization_factor(p, 0, "bogus")
    out = ctypes.c_double()
    with pytest.raises(ValueError):
        N.check(N.lib().mbs_normalization_factor(10, 4, 0, 7, ctypes.byref(out)))


def test_plan_validation_matches_reference():
    with pytest.raises(ValueError):
        mbs.MicroBatchPlan(n_b=10, n_mu=4, n_s_mu=2, sizes=(4, 4), index_ranges=((0, 4), (4, 8)))
    with pytest.raises(ValueError):
        mbs.MicroBatchPlan(n_b=8, n_mu=4, n_s_mu=2, sizes=(5, 3), index_ranges=((0, 5), (5, 8)))


def test_host_gather_native():
    rs = np.random.RandomState(0)
    x = rs.randint(0, 255, size=(97, 3, 5, 7), dtype=np.uint8)
    rows = rs.permutation(97)[:41].astype(np.int64)
    out = np.empty((41, 3, 5, 7), dtype=np.uint8)
    for threads in (1, 3, 8):
        out[:] = 0
        N.check(N.lib().mbs_host_gather(x.ctypes.data, x[0].nbytes, rows.ctypes.data, len(rows), out.ctypes.data,
                                        threads))
        assert np.array_equal(out, x[rows])
    big = rs.randn(300, 9000)
    r2 = rs.randint(0, 300, size=500).astype(np.int64)
    o2 = np.empty((500, 9000))
    N.check(N.lib().mbs_host_gather(big.ctypes.data, big[0].nbytes, r2.ctypes.data, 500, o2.ctypes.data, 8))
    assert np.array_equal(o2, big[r2])


def test_status_mapping():
    assert N.lib().mbs_status_string(2) == b"accumulator overflow"
    with pytest.raises(mbs.AccumulatorOverflowError):
        N.check(N.EOVERFLOW)
    with pytest.raises(mbs.GradientKeyMismatchError):
        N.check(N.EKEY)
    with pytest.raises(mbs.NonFiniteError):
        N.check(N.ENONFINITE)
    with pytest.raises(RuntimeError):
        N.check(N.ECUDA)


def test_rng_matches_reference_fixtures():
    g = load_json("rng.json")
    for k, h in g["keys"].items():
        seed, name = k.split("|", 1)
        assert hex(mbs.stream_key(int(seed), name)) == h
    for k, perm in g["perms"].items():
        seed, epoch, n = map(int, k.split("|"))
        assert mbs.epoch_order(n, seed, epoch).tolist() == perm


def test_linear_lr_matches_reference():
    g = load_json("misc.json")
    for lr0, s, tot, h in g["linear_lr"]:
        assert mbs.linear_lr(lr0, s, tot).hex() == h
    with pytest.raises(ValueError):
        mbs.linear_lr(0.1, 11, 10)
