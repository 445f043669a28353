"""Tensor-core (tcgen05 kind::tf32) screening scan: error model and parity.

The TC scan only SCREENS: every key it stores must be a rigorous lower bound of
the exact scipy-order FP64 value (nnm_tc.cu header).  The probe runs the real
kernel on chosen tile pairs, dumps the accumulators and checks every pair:
no key above its exact value, and |v - S| well inside the bound that the keys
are built from (which validates the tensor-core accumulation constant).
Parity: the clustering with the TC scan equals the oracle and the FP32 path.
All @gpu.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from nnm_testutil import ROOT

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _general_path(monkeypatch):
    """These tests exercise the tile / tensor-core path: keep small inputs off the
    single-launch small-input kernel."""
    monkeypatch.setenv("NNM_SMALL", "0")

FIELDS = ("root_a", "root_b", "dist", "new_size", "point_a", "point_b")


@pytest.fixture(scope="module")
def nnm():
    import paper_1402_3789_b200 as pkg
    from paper_1402_3789_b200 import _native

    _native.load()
    return pkg


def _tiles(lib, dd):
    tp, rows = ctypes.c_int64(), ctypes.c_int64()
    from paper_1402_3789_b200 import _native

    _native.check(lib.nnm_bv_begin(dd.handle, 0, np.nan, ctypes.byref(tp), ctypes.byref(rows)))
    T = int((math.isqrt(8 * tp.value + 1) - 1) // 2)
    assert T * (T + 1) // 2 == tp.value
    return T


@pytest.mark.parametrize("shape", [(20000, 25, 40, 1.0), (6000, 8, 12, 1.0), (5000, 25, 5, 0.01),
                                   (4000, 29, 8, 30.0)])
def test_tc_error_model_probe(nnm, shape):
    from paper_1402_3789_b200 import _native

    n, d, k, spread = shape
    X = nnm.generate_synthetic(n, d, k, spread, seed=17)[0]
    lib = _native.load()
    dd = _native.DeviceDataset(X)
    T = _tiles(lib, dd)
    rng = np.random.default_rng(5)
    items = [(i, i) for i in range(0, T, 3)]
    items += [(i, i + 1) for i in range(0, T - 1, 2)]
    items += [(int(a), int(b)) for a, b in rng.integers(0, T, size=(200, 2))]
    items = np.array(items[:600], dtype=np.int32)
    out = (ctypes.c_double * 3)()
    _native.check(lib.nnm_tc_probe(dd.handle, items.ctypes.data, len(items), out))
    worst, bad, cnt = out[0], int(out[1]), int(out[2])
    assert cnt > 100_000
    assert bad == 0, f"{bad} keys above their exact value"
    assert worst < 0.9, f"evaluation error reaches {worst:.3f} of the bound"


def test_tc_probe_rejects_bad_input(nnm):
    from paper_1402_3789_b200 import _native

    X = nnm.generate_synthetic(500, 40, 3, 1.0, seed=1)[0]
    dd = _native.DeviceDataset(X)
    out = (ctypes.c_double * 3)()
    items = np.zeros(2, np.int32)
    rc = _native.load().nnm_tc_probe(dd.handle, items.ctypes.data, 1, out)
    assert rc == _native.NNM_E_UNSUPPORTED


def _run_env(code: str, env_extra: dict) -> str:
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout


@pytest.mark.parametrize("kind", ["blobs", "shuffled", "ties", "dmax"])
def test_tc_path_vs_oracle(nnm, kind):
    """The default (TC) Euclidean Boruvka path against the C oracle, bit-exact."""
    from oracle import nnm_oracle as orc

    rng = np.random.default_rng(11)
    cons = {}
    if kind == "blobs":
        X = nnm.generate_synthetic(4000, 25, 17, 1.0, seed=3)[0]
    elif kind == "shuffled":
        X = nnm.generate_synthetic(4000, 12, 9, 2.0, seed=4)[0]
        X = X[rng.permutation(len(X))]
    elif kind == "ties":
        X = rng.integers(-3, 4, size=(3000, 6)).astype(np.float64)
    else:
        X = nnm.generate_synthetic(4000, 25, 20, 1.0, seed=6)[0]
        cons = {"dmax": 5.0}
    res = nnm.fit(X, **cons)
    assert res.device_stats["tc_items"] > 0
    m_or, a_or = orc.single_linkage(X, **cons)
    got = res.merges.array
    assert len(got) == len(m_or)
    for f in FIELDS:
        assert np.array_equal(got[f], m_or[f]), f
    assert np.array_equal(res.assignments, a_or)


def test_tc_and_fp32_paths_identical_at_scale(nnm):
    """60k x 25 blobs: the TC scan and the FP32 dot-form scan give the same dendrogram
    (run in subprocesses: the path is chosen per process by NNM_TC)."""
    code = ("import numpy as np, hashlib, paper_1402_3789_b200 as nnm\n"
            "X = nnm.generate_synthetic(60000, 25, 120, 1.0, seed=9)[0]\n"
            "r = nnm.fit(X)\n"
            "print(hashlib.sha256(r.merges.array.tobytes() + r.assignments.tobytes()).hexdigest(),"
            " r.device_stats['tc_items'] > 0)\n")
    a = _run_env(code, {"NNM_TC": "1"}).split()
    b = _run_env(code, {"NNM_TC": "0"}).split()
    assert a[1] == "True" and b[1] == "False"
    assert a[0] == b[0]


@pytest.mark.parametrize("cfg", ["c4", "c3"])
def test_tile_pair_bound_cache_identical_at_full_scale(nnm, cfg):
    """BASELINE configs 4 (2M x 25 full dendrogram) and 3 (500k x 25, dmax=5): the
    tile-pair lower-bound cache (phase-2 pairs pruned with bounds from earlier scans)
    gives byte-identical merges and labels to the scan without it, and scans fewer
    tile pairs."""
    code = ("import hashlib, paper_1402_3789_b200 as nnm\n"
            "from paper_1402_3789_b200.datagen import config_dataset\n"
            f"X = config_dataset('{cfg}')\n"
            f"r = nnm.fit(X, dmax={'5.0' if cfg == 'c3' else 'None'})\n"
            "print(hashlib.sha256(r.merges.array.tobytes() + r.assignments.tobytes()).hexdigest(),"
            " r.device_stats['tc_items'], len(r.merges))\n")
    a = _run_env(code, {"NNM_TPCACHE": "1"}).split()
    b = _run_env(code, {"NNM_TPCACHE": "0"}).split()
    assert a[0] == b[0]
    assert a[2] == b[2]
    if cfg == "c4":
        assert a[2] == "1999999"
        assert int(a[1]) < int(b[1])


def test_tc_deferred_and_in_epilogue_keys_identical(nnm):
    """500k x 25 (config 3's data, no dmax): phase-1 exact keys evaluated after the scan
    from the appended candidates (default) and inside the epilogue (NNM_TC_DEFER=0) give
    byte-identical dendrograms."""
    code = ("import hashlib, paper_1402_3789_b200 as nnm\n"
            "from paper_1402_3789_b200.datagen import config_dataset\n"
            "X = config_dataset('c3')\n"
            "r = nnm.fit(X)\n"
            "print(hashlib.sha256(r.merges.array.tobytes() + r.assignments.tobytes()).hexdigest(),"
            " r.device_stats['tc_items'] > 0, len(r.merges))\n")
    a = _run_env(code, {"NNM_TC_DEFER": "1"}).split()
    b = _run_env(code, {"NNM_TC_DEFER": "0"}).split()
    assert a[1] == "True" and b[1] == "True"
    assert a[0] == b[0] and a[2] == b[2] == "499999"


@pytest.mark.parametrize("metric", ["manhattan", "chebyshev"])
def test_fp32_tile_pair_cache_identical(nnm, metric):
    """500k x 25, L1 / L-inf: the FP32 direct scan's tile-pair cache (exact_lower of each
    item's minimum) prunes later rounds without changing the dendrogram."""
    code = ("import hashlib, paper_1402_3789_b200 as nnm\n"
            "from paper_1402_3789_b200.datagen import config_dataset\n"
            "X = config_dataset('c3')\n"
            f"r = nnm.fit(X, metric='{metric}')\n"
            "print(hashlib.sha256(r.merges.array.tobytes() + r.assignments.tobytes()).hexdigest(),"
            " int(r.device_stats['pairs_evaluated']))\n")
    a = _run_env(code, {"NNM_TPCACHE": "1"}).split()
    b = _run_env(code, {"NNM_TPCACHE": "0"}).split()
    assert a[0] == b[0]
    assert int(a[1]) < int(b[1])
