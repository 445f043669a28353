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
    every byte of assignments.csv / merges.csv matches; on the default Boruvka path
    (no kl2/kl3/kl4) everything but the P-dependent round column matches."""
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
        round_path = exact_rounds or any(f in case["flags"] for f in ("--kl2", "--kl3", "--kl4"))
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
