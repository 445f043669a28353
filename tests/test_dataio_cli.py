"""dataio + CLI drop-in against the reference's own outputs.

Golden fixtures (tests/golden/cli_cases.json) were produced by the reference
(tests/golden/make_cli_golden.py): load_dataset outcomes on edge-case CSVs and
the exact assignments.csv / merges.csv / stats.json of `parclust cluster` runs.
CPU tests pin the parser, the writers and replay_merges; @gpu tests run the
GPU CLI end to end and compare the files byte for byte.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from nnm_testutil import GOLDEN

FIELDS_NO_ROUND = ("step", "root_a", "root_b", "distance", "new_size")


@pytest.fixture(scope="module")
def golden():
    return json.load(open(os.path.join(GOLDEN, "cli_cases.json")))


def test_load_dataset_matches_reference(golden, tmp_path):
    from paper_1402_3789_b200.dataio import load_dataset
    from paper_1402_3789_b200.model import ValidationError

    for name, case in golden["parse"].items():
        path = tmp_path / f"{name}.csv"
        path.write_text(case["text"], encoding="utf-8")
        if "error" in case:
            with pytest.raises(ValidationError) as ei:
                load_dataset(str(path), id_column=case["id_column"])
            assert str(ei.value).replace(str(path), "<path>") == case["error"], name
        else:
            ds = load_dataset(str(path), id_column=case["id_column"])
            assert ds.values.tolist() == case["values"], name
            assert [str(v) for v in ds.ids.tolist()] == case["ids"], name


def _parse_outputs(case):
    ids_lines = case["assignments"].splitlines()[1:]
    ids = [ln.split(",")[0] for ln in ids_lines]
    pos = {v: i for i, v in enumerate(ids)}
    assign = np.array([pos[ln.split(",")[1]] for ln in ids_lines], dtype=np.int64)
    rows = [ln.split(",") for ln in case["merges"].splitlines()[1:]]
    return ids, assign, rows


def _result_from_golden(case):
    from paper_1402_3789_b200.engine import RunResult
    from paper_1402_3789_b200.model import MergeEvent
    from paper_1402_3789_b200.scheduler import UtilizationStats

    ids, assign, rows = _parse_outputs(case)
    merges = [MergeEvent(step=int(r[0]), round=int(r[1]), root_a=int(r[2]), root_b=int(r[3]),
                         dist=float(r[4]), new_size=int(r[5]), point_a=-1, point_b=-1)
              for r in rows]
    st = case["stats"]
    return RunResult(merges=merges, assignments=assign, rounds=st["rounds"],
                     stop_reason=st["stop_reason"], stats=UtilizationStats(),
                     round_counters=st["round_counters"])


def test_write_outputs_bytes_match_reference(golden, tmp_path):
    from paper_1402_3789_b200.dataio import load_dataset, write_outputs

    for name, case in golden["runs"].items():
        inp = tmp_path / f"{name}.csv"
        inp.write_text(case["input"], encoding="utf-8")
        ds = load_dataset(str(inp), id_column="id" if case["with_ids"] else None)
        res = _result_from_golden(case)
        paths = write_outputs(res, str(tmp_path / name), dataset=ds,
                              config_echo=case["stats"]["config"])
        assert open(paths["assignments"]).read() == case["assignments"], name
        assert open(paths["merges"]).read() == case["merges"], name
        st = json.load(open(paths["stats"]))
        for k, v in case["stats"].items():
            assert st[k] == v, (name, k)


def test_replay_merges_matches_reference_assignments(golden):
    from paper_1402_3789_b200.dataio import replay_merges

    for name, case in golden["runs"].items():
        ids, assign, rows = _parse_outputs(case)
        got = replay_merges(len(ids), [(int(r[2]), int(r[3])) for r in rows])
        assert np.array_equal(got, assign), name


def test_cli_validation_exit_codes(tmp_path, capsys):
    from paper_1402_3789_b200.cli import main

    assert main(["cluster"]) == 1
    assert "--input is required" in capsys.readouterr().err
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("pairs-per-batch = 8\nbogus = 1\n")
    assert main(["cluster", "--config", str(cfg), "--input", "x.csv"]) == 1
    assert "unknown setting 'bogus'" in capsys.readouterr().err
    assert main(["cluster", "--input", str(tmp_path / "missing.csv")]) == 1
    assert main(["cluster", "--input", "x.csv", "--metric", "cosine"]) == 1
    assert main(["frobnicate"]) == 1


def test_cli_generate_round_trips(tmp_path):
    from paper_1402_3789_b200.cli import main
    from paper_1402_3789_b200.datagen import generate_synthetic
    from paper_1402_3789_b200.dataio import load_dataset

    out = tmp_path / "blobs.csv"
    assert main(["generate", "--out", str(out), "--n", "300", "--d", "4", "--clusters", "3",
                 "--spread", "0.5", "--seed", "9"]) == 0
    X, labels = generate_synthetic(300, 4, 3, 0.5, 9)
    assert np.array_equal(load_dataset(str(out)).values, X)  # %.17g round trip, bit-exact
    assert np.array_equal(np.loadtxt(tmp_path / "blobs.labels.csv", dtype=np.int64), labels)


@pytest.mark.gpu
@pytest.mark.parametrize("exact_rounds", [True, False])
def test_cli_cluster_matches_reference_bytes(golden, tmp_path, exact_rounds):
    """GPU CLI vs the reference CLI on the same input and flags.  With --exact-rounds
    every byte of assignments.csv / merges.csv matches (also with kl4); otherwise (the
    Boruvka path, or kl2/kl3 in large batches) everything but the P-dependent round column
    matches."""
    from paper_1402_3789_b200.cli import main

    for name, case in golden["runs"].items():
        inp = tmp_path / f"{name}.csv"
        inp.write_text(case["input"], encoding="utf-8")
        od = tmp_path / f"out_{name}_{exact_rounds}"
        argv = ["cluster", "--input", str(inp), "--out-dir", str(od)] + case["flags"]
        if case["with_ids"]:
            argv += ["--id-column", "id"]
        if exact_rounds:
            argv.append("--exact-rounds")
        assert main(argv) == 0, name
        assert (od / "assignments.csv").read_text() == case["assignments"], name
        got = (od / "merges.csv").read_text()
        st = json.load(open(od / "stats.json"))
        # rounds (and the per-round skip counters) are part of the result only with kl4
        # or --exact-rounds; kl2/kl3 alone run large GPU batches
        round_path = exact_rounds or "--kl4" in case["flags"]
        if round_path:
            assert got == case["merges"], name
            for k, v in case["stats"].items():
                assert st[k] == v, (name, k)
        else:
            drop = lambda text: [",".join(r.split(",")[:1] + r.split(",")[2:])  # noqa: E731
                                 for r in text.splitlines()]
            assert drop(got) == drop(case["merges"]), name
            for k in ("config", "n", "d", "merges", "final_clusters", "stop_reason"):
                assert st[k] == case["stats"][k], (name, k)


def _native_available():
    from nnm_testutil import ROOT

    return os.path.exists(os.path.join(ROOT, "paper_1402_3789_b200", "libnnm.so"))


_TOKENS_OK = ["0", "1", "-1", "+2", "3.25", ".5", "5.", "1e5", "1E-5", "-1e+02", "1_000",
              "2.5_5", "6e1_0", "123456789012345678901234567890", "0.1", "1e-320", "9.999e307",
              "-0.0", "4_4.0_1"]
_TOKENS_BAD = ["abc", "1__0", "_1", "1_", "0x10", "1e", "e5", "--1", "1.2.3", "", "1 2", "nan",
               "-inf", "Infinity", "1e999"]
_WS = ["", " ", "\t", " ", "　", "  "]
_EOL = ["\n", "\r\n", "\r", "\x0b", "\x0c", "\x1c", " "]


@pytest.mark.skipif(not _native_available(), reason="libnnm.so not built")
def test_native_csv_fuzz_matches_restatement(tmp_path):
    """nnm_csv_load (C++) vs the line-by-line restatement of dataio.py:49-116 on random
    files: identical values (bitwise), ids and error messages."""
    from paper_1402_3789_b200.dataio import _load_dataset_py, load_dataset
    from paper_1402_3789_b200.model import ValidationError

    rng = np.random.default_rng(1234)
    for case in range(300):
        ncols = int(rng.integers(1, 6))
        rows = int(rng.integers(1, 40))
        lines = []
        header = rng.random() < 0.3
        if header:
            lines.append(",".join(f"c{j}" for j in range(ncols)))
        for _ in range(rows):
            toks = []
            for _ in range(ncols):
                pool = _TOKENS_BAD if rng.random() < 0.01 else _TOKENS_OK
                t = pool[int(rng.integers(len(pool)))]
                toks.append(_WS[int(rng.integers(len(_WS)))] + t + _WS[int(rng.integers(len(_WS)))])
            if rng.random() < 0.02:
                toks = toks[:-1] if len(toks) > 1 else toks + ["1"]
            lines.append(",".join(toks))
            if rng.random() < 0.05:
                lines.append(_WS[int(rng.integers(len(_WS)))])
        text = "".join(ln + _EOL[int(rng.integers(len(_EOL)))] for ln in lines)
        path = tmp_path / f"f{case}.csv"
        path.write_bytes(text.encode("utf-8"))
        idc = None
        if header and rng.random() < 0.5:
            idc = "c0" if rng.random() < 0.5 else str(int(rng.integers(0, ncols + 1)))
        outs = []
        for fn in (load_dataset, _load_dataset_py):
            try:
                ds = fn(str(path), id_column=idc)
                outs.append(("ok", ds.values.tobytes(), ds.values.shape, [str(v) for v in ds.ids.tolist()]))
            except ValidationError as exc:
                outs.append(("err", str(exc)))
        assert outs[0] == outs[1], (case, text[:200], outs[0][:1], outs[1][:1])


@pytest.mark.skipif(not _native_available(), reason="libnnm.so not built")
def test_native_csv_large_round_trip(tmp_path):
    """200k x 25 written as %.17g parses back bit-exactly through the native loader."""
    import time

    from paper_1402_3789_b200.datagen import generate_synthetic
    from paper_1402_3789_b200.dataio import Dataset, load_dataset, write_dataset

    X = generate_synthetic(200_000, 25, 400, 1.0, seed=3)[0]
    path = tmp_path / "big.csv"
    write_dataset(Dataset(values=X), str(path))
    t0 = time.perf_counter()
    ds = load_dataset(str(path))
    dt = time.perf_counter() - t0
    assert np.array_equal(ds.values, X)
    assert dt < 10.0  # the Python loop takes ~12 s here
