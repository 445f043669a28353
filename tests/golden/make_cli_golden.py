"""Generate golden fixtures for the dataio / CLI drop-in (run in the build container,
where the reference is importable):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Writes tests/golden/cli_cases.json:
* "parse": CSV texts with the reference's load_dataset outcome (values + ids, or
  the ValidationError message with the file path replaced by "<path>");
* "runs":  input CSV texts, the reference CLI flags, and the exact contents of the
  reference's assignments.csv / merges.csv plus the deterministic stats.json keys.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from parclust import cli, dataio  # noqa: E402  (reference, via PYTHONPATH)
from parclust.model import ValidationError  # noqa: E402

PARSE_CASES = {
    "plain": "1,2,3\n4,5,6\n",
    "header": "a,b,c\n1,2,3\n4.5,-6e-3,7\n",
    "blank_lines": "\n1,2\n\n3,4\n   \n5,6\n",
    "id_by_name": "id,x,y\np1,0.5,1\np2,1.5,2\n",
    "id_by_index": "x,name,y\n1,q,2\n3,r,4\n",
    "ragged": "1,2,3\n4,5\n",
    "non_numeric": "x,y\n1,2\n3,abc\n",
    "non_finite": "1,2\nnan,3\n",
    "inf": "1,inf\n",
    "empty": "\n\n",
    "header_only": "a,b\n",
    "dup_id": "id,x\nk,1\nk,2\n",
    "bad_id_name": "a,b\n1,2\n",
    "id_index_out_of_range": "1,2\n3,4\n",
    "spaces": " 1 , 2 \n 3 ,4\n",
    "underscores": "1_000,2.5_5\n3e1_0,-_4\n",
    "underscores_ok": "1_000,2.5_5\n3e1_0,4_4.0_1\n",
    "bad_underscore": "1__0,2\n",
    "inf_words": "INF,-Infinity\n",
    "nan_word": "1,NaN\n",
    "hex": "0x10,1\n",
    "exp_forms": "1E5,.5\n5.,-1e-3\n+2,1e+02\n",
    "crlf_cr": "1,2\r\n3,4\r5,6\r\n",
    "vt_ff_seps": "1,2\x0b3,4\x0c5,6\x1c7,8\n",
    "unicode_space": "\u00a01,2\u2003\n3,\u30004\n",
    "tabs": "\t1\t,2\n3,4\t\n",
    "quote_token": "1,2\n3,it's\n",
    "id_index_str": "a,b,c\n1,2,3\n4,5,6\n",
    "id_index_padded": "1,2,3\n4,5,6\n",
    "id_index_neg": "1,2\n3,4\n",
    "id_header_numeric_name": "x,1,y\n5,p,6\n7,q,8\n",
    "header_mixed": "1,b,3\n4,5,6\n",
    "trailing_delim": "1,2,\n3,4,\n",
    "empty_field": "1,,3\n",
    "semicolons_in_field": "1;2,3\n",
}
PARSE_ID = {"id_by_name": "id", "id_by_index": "1", "dup_id": "id", "bad_id_name": "zz",
            "id_index_out_of_range": "5", "id_index_str": "2", "id_index_padded": " 01 ",
            "id_index_neg": "-1", "id_header_numeric_name": "1"}


def parse_cases(tmp):
    out = {}
    for name, text in PARSE_CASES.items():
        path = os.path.join(tmp, f"{name}.csv")
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
        try:
            ds = dataio.load_dataset(path, id_column=PARSE_ID.get(name))
            out[name] = {"text": text, "id_column": PARSE_ID.get(name),
                         "values": ds.values.tolist(), "ids": [str(v) for v in ds.ids.tolist()],
                         "ids_are_default": name not in PARSE_ID}
        except ValidationError as exc:
            out[name] = {"text": text, "id_column": PARSE_ID.get(name),
                         "error": str(exc).replace(path, "<path>")}
    return out


def csv_text(X, ids=None):
    rows = []
    if ids is not None:
        rows.append("id," + ",".join(f"f{k}" for k in range(X.shape[1])))
    for i, row in enumerate(X):
        vals = ",".join("%.17g" % v for v in row)
        rows.append(f"{ids[i]},{vals}" if ids is not None else vals)
    return "\n".join(rows) + "\n"


RUNS = [
    # (name, dataset builder, CLI flags)
    ("blobs_ids_P64", lambda: dataio.generate_synthetic(600, 5, 7, 1.0, 21), True,
     ["--pairs-per-batch", "64", "--seed", "3"]),
    ("constrained_kl", lambda: dataio.generate_synthetic(500, 4, 9, 2.0, 22), False,
     ["--pairs-per-batch", "32", "--kl1", "6", "--kl2", "60", "--kl3", "90", "--kl4", "20"]),
    ("manhattan_dmax", lambda: dataio.generate_synthetic(400, 3, 5, 1.5, 23), False,
     ["--metric", "manhattan", "--dmax", "2.5", "--pairs-per-batch", "128"]),
]
STATS_KEYS = ("config", "n", "d", "rounds", "merges", "final_clusters", "stop_reason", "skips",
              "round_counters")


def run_cases(tmp):
    out = {}
    for name, build, with_ids, flags in RUNS:
        ds, _ = build()
        ids = [f"pt{i:04d}" for i in range(ds.n)] if with_ids else None
        text = csv_text(ds.values, ids)
        path = os.path.join(tmp, f"{name}.csv")
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
        od = os.path.join(tmp, name)
        argv = ["cluster", "--input", path, "--out-dir", od] + (["--id-column", "id"] if with_ids else []) + flags
        rc = cli.main(argv)
        assert rc == 0, (name, rc)
        stats = json.load(open(os.path.join(od, "stats.json")))
        out[name] = {"input": text, "flags": flags, "with_ids": with_ids,
                     "assignments": open(os.path.join(od, "assignments.csv")).read(),
                     "merges": open(os.path.join(od, "merges.csv")).read(),
                     "stats": {k: stats[k] for k in STATS_KEYS}}
    return out


def main():
    with tempfile.TemporaryDirectory() as tmp:
        payload = {"parse": parse_cases(tmp), "runs": run_cases(tmp)}
    with open(os.path.join(HERE, "cli_cases.json"), "w", encoding="utf-8") as fh:
        json.dump(payload, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print("wrote", os.path.join(HERE, "cli_cases.json"))


if __name__ == "__main__":
    sys.exit(main())
