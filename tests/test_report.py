"""RunReport parity (cli.py:68-221): the GPU run() against the
reference's own cli.run reports (tests/golden/make_golden_report.py): same
schema and integer fields, front-statistics CSV identical, iterations within
one, residuals alike."""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _fixture():
    with open(os.path.join(HERE, "golden", "report.json")) as fh:
        return json.load(fh)


def test_config_validation_and_labels():
    from paper_1410_2697_b200.report import RunConfig, mode_label, parse_generator
    with pytest.raises(ValueError, match="exactly one of --matrix or --gen is required"):
        RunConfig().validate()
    with pytest.raises(ValueError, match="unknown mode 'x'"):
        RunConfig(generator="poisson:2,2,2", mode="x").validate()
    with pytest.raises(ValueError, match="unknown preconditioner 'y'"):
        RunConfig(generator="poisson:2,2,2", precond="y").validate()
    with pytest.raises(ValueError, match="expected poisson:NX,NY,NZ"):
        parse_generator("poisson:2,2")
    A, b = parse_generator("poisson:3,4,5")
    assert A.n_rows == 60 and np.array_equal(b, np.ones(60))
    assert mode_label(RunConfig(mode="gmres", precond="ilut")) == "gmres+ilut"
    assert mode_label(RunConfig(mode="amf")) == "direct-accelerated"


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(_fixture()))
def test_report_matches_reference(tmp_path, name):
    from paper_1410_2697_b200.report import RunConfig, run
    fx = _fixture()[name]
    out = str(tmp_path / f"{name}.json")
    rep = run(RunConfig(out=out, **fx["config"]))
    d = json.load(open(out))
    ref = fx["report"]
    assert set(d) - {"factor_time_s", "solve_time_s", "history_csv", "front_stats_csv"} == set(ref)
    for k in ("n", "nnz", "mode", "peak_stored_reals"):
        assert d[k] == ref[k], k
    if "iterations" in ref:
        assert abs(d["iterations"] - ref["iterations"]) <= 1
        assert d["final_relative_residual"] <= 10 * max(ref["final_relative_residual"], 1e-12)
        hist = open(d["history_csv"]).read().splitlines()
        assert hist[0] == "iteration,relative_residual" and abs(len(hist) - len(fx["side"]["history_csv"].splitlines())) <= 1
    else:
        assert np.isclose(d["final_relative_residual"], ref["final_relative_residual"], rtol=1e-3, atol=1e-13)
    if "front_stats_csv" in fx["side"]:
        assert open(d["front_stats_csv"]).read() == fx["side"]["front_stats_csv"]
    assert rep.to_dict()["mode"] == ref["mode"]
