"""The harness CLI (`python -m paper_2112_15198_b200 run/verify/scale`,
tools/ifgf.cpp) on the B200: the JSON report of schema 1, results equal to
the unmodified reference's apply on the same cube-face surface, the comm
statistics of `--ranks` equal to the reference's run_distributed counters,
verify's exit codes and scale's CSV."""
import argparse
import csv
import io
import json

import numpy as np
import pytest

from paper_2112_15198_b200 import cli

pytestmark = pytest.mark.gpu


def _opts(cmd, *args):
    p = argparse.ArgumentParser()
    sub = p.add_subparsers(dest="cmd")
    cli.add_common(sub.add_parser(cmd))
    return p.parse_args([cmd, *args])


def test_run_report_schema_1(gpu, tmp_path):
    out = tmp_path / "r.json"
    assert cli.main(["run", "--n", "3000", "--size-lambda", "3", "--seed", "5",
                     "--output", str(out)]) == 0
    j = json.loads(out.read_text())
    assert j["schema_version"] == 1
    for k in ("config", "n", "depth", "diameter_lambda", "h_level_d_lambda", "stage_seconds",
              "epsilon", "levels", "peak_live_blocks", "simd_variant", "result_checksum",
              "imag_max_abs"):
        assert k in j, k
    assert j["n"] == 6 * 22 * 22
    assert abs(j["diameter_lambda"] - 3.0) < 1e-12
    assert j["epsilon"]["m"] == 1000 and j["epsilon"]["value"] <= 5e-3
    assert len(j["result_checksum"]) == 16
    assert [l["d"] for l in j["levels"]] == list(range(3, j["depth"] + 1))


def test_run_matches_reference_apply(gpu, ref):
    o = _opts("run", "--n", "3000", "--size-lambda", "3", "--seed", "5")
    b = cli.build_case(o)
    cli._evaluate(b, 1)
    from bindings import Params
    want_re, want_im, _ = ref.apply(b.pc.x1, b.pc.x2, b.pc.x3, b.pc.a_re, b.pc.a_im, 0,
                                    b.cfg.wavenumber, Params(threads=4))
    err = np.sqrt(np.sum((b.pc.i_re - want_re) ** 2 + (b.pc.i_im - want_im) ** 2) /
                  np.sum(want_re ** 2 + want_im ** 2))
    assert err <= 1e-10


@pytest.mark.parametrize("ranks", [2, 4])
def test_ranks_comm_stats_match_reference(gpu, ref, ranks):
    o = _opts("run", "--n", "6000", "--size-lambda", "4", "--seed", "3", "--ranks", str(ranks))
    b = cli.build_case(o)
    _, comm = cli._evaluate(b, ranks)
    got = b.pc.i_re.copy(), b.pc.i_im.copy()
    b1 = cli.build_case(o)
    cli._evaluate(b1, 1)
    assert np.array_equal(got[0], b1.pc.i_re) and np.array_equal(got[1], b1.pc.i_im)
    from bindings import Params
    _, _, rc = ref.run_distributed(b.pc.x1, b.pc.x2, b.pc.x3, b.pc.a_re, b.pc.a_im, 0,
                                   b.cfg.wavenumber, Params(threads=4), ranks)
    keys = ["interp_fetched", "prop_fetched", "max_interp_fanout", "max_prop_fanout",
            "owned_blocks", "peak_rank_cache_blocks"]
    for row, lev in zip(rc, comm.levels):
        assert [int(row[i]) for i in range(6)] == [lev[k] for k in keys], (lev, row)
    assert comm.total_fetched() == int(rc[:, 0].sum() + rc[:, 1].sum())


def test_verify_exit_codes(gpu, capsys):
    assert cli.main(["verify", "--n", "2000", "--size-lambda", "2"]) == 0
    assert "pass" in capsys.readouterr().out
    assert cli.main(["verify", "--n", "2000", "--size-lambda", "2", "--threshold", "1e-12"]) == 1
    assert "FAIL" in capsys.readouterr().out
    assert cli.main(["verify", "--n", "1500", "--size-lambda", "2", "--verify", "full"]) == 0
    assert cli.main(["verify", "--n", "4000", "--size-lambda", "2", "--ranks", "2"]) == 0
    assert cli.main(["verify", "--n", "6000", "--verify", "full"]) == 2  # N <= 5000 only


def test_scale_csv(gpu, tmp_path):
    out = tmp_path / "s.csv"
    assert cli.main(["scale", "--ns", "2000,8000", "--size-lambda", "2",
                     "--output", str(out)]) == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert len(rows) == 2
    assert list(rows[0]) == ["n", "size_lambda", "depth", "t_seconds", "t_per_nlog2n",
                             "peak_live_blocks", "relevant_cones", "blocks_fetched_total",
                             "fetched_per_nlog2n"]
    assert abs(float(rows[1]["size_lambda"]) - 4.0) < 1e-9  # fixed points per box
