"""Fixture for RunReport parity (cli.py:68-221): the REFERENCE's cli.run on
small problems; the JSON reports (times dropped) and the side CSVs.

    MFH_REF_SRC=/tmp/refbuild/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_report.py
"""
import json
import os
import sys
import tempfile

REF = os.environ.get("MFH_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))

from mfhodlr import cli  # noqa: E402

RUNS = {
    "amf": dict(generator="poisson:9,8,7", mode="amf", n_c=48, eps=1e-6, d=1, n_leaf=16, leaf_size=32),
    "mf": dict(generator="poisson:6,6,6", mode="mf", leaf_size=16),
    "gmres_amf": dict(generator="poisson:9,8,7", mode="gmres", precond="amf", n_c=48, eps=1e-3, d=1, n_leaf=16,
                      leaf_size=32, tol=1e-10, restart=30),
    "gmres_ilut": dict(generator="poisson:8,8,8", mode="gmres", precond="ilut", k=2, drop_tol=1e-3, tol=1e-10,
                       restart=30),
    "gmres_diag_scaled": dict(generator="poisson:6,5,4", mode="gmres", precond="diag", tol=1e-10, restart=20,
                              scale_rows=True),
}
out = {}
with tempfile.TemporaryDirectory() as td:
    for name, kw in RUNS.items():
        path = os.path.join(td, name + ".json")
        rep = cli.run(cli.RunConfig(out=path, **kw))
        d = rep.to_dict()
        side = {}
        for key in ("history_csv", "front_stats_csv"):
            if key in d:
                side[key] = open(d[key]).read()
        for key in ("factor_time_s", "solve_time_s", "history_csv", "front_stats_csv"):
            d.pop(key, None)
        out[name] = {"config": kw, "report": d, "side": side}
        print(name, d)
json.dump(out, open(os.path.join(HERE, "report.json"), "w"), indent=1, sort_keys=True)
