"""The reference's harness around the operator (§8(f) "harness
compatibility"): cube-face surfaces (geometry.cpp:57-93), the IFGF v1 binary
and CSV point formats (geometry.cpp:147-226), checksum_hex (bench.cpp:26-41)
and the `ifgf run/verify/scale` CLI front end (tools/ifgf.cpp).  Pinned
against the unmodified reference (oracle/_ref) where it is built; no GPU."""
import json
import os

import numpy as np
import pytest

from paper_2112_15198_b200 import cli, points


@pytest.mark.parametrize("shape,npd,seed", [(0, 2, 1), (0, 9, 7), (1, 5, 3), (2, 4, 11)])
def test_generate_surface_bitwise_equal_to_reference(ref, shape, npd, seed):
    pc = points.generate_surface(shape, 1.0, npd, seed)
    want = ref.generate_surface(shape, 1.0, npd, seed)
    for got, w in zip((pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im), want):
        assert np.array_equal(got, w)


def test_generate_surface_structure():
    pc = points.generate_surface(0, 2.0, 6, 5)
    assert pc.size() == 6 * 36
    r = np.sqrt(pc.x1 ** 2 + pc.x2 ** 2 + pc.x3 ** 2)
    assert np.allclose(r, 2.0, rtol=0, atol=1e-14)
    assert (pc.a_re >= 0).all() and (pc.a_re < 1).all()
    prol = points.generate_surface(2, 1.0, 6, 5)
    assert np.allclose(prol.x3, 10.0 * pc.x3 / 2.0, rtol=0, atol=1e-13)
    with pytest.raises(Exception):
        points.generate_surface(0, 1.0, 1, 5)  # n_per_dim >= 2 (geometry.cpp:59)
    with pytest.raises(Exception):
        points.generate_surface(0, -1.0, 4, 5)  # a > 0 (geometry.cpp:58)


def test_checksum_matches_reference(ref):
    rng = np.random.default_rng(3)
    re, im = rng.standard_normal(1001), rng.standard_normal(1001)
    assert points.checksum_hex(re, im) == ref.checksum_hex(re, im)
    assert points.checksum_hex(np.zeros(0), np.zeros(0)) == ref.checksum_hex(np.zeros(0), np.zeros(0))


def test_binary_format_round_trips_with_reference(ref, tmp_path):
    pc = points.generate_surface(1, 1.0, 7, 2)
    ours = tmp_path / "ours.ifgf"
    points.write_points_binary(str(ours), pc)
    back = ref.read_points(ours)  # the reference reads our file
    for got, w in zip(back, (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)):
        assert np.array_equal(got, w)
    theirs = tmp_path / "theirs.ifgf"
    ref.write_points_binary(theirs, pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)
    assert theirs.read_bytes() == ours.read_bytes()  # byte-identical files
    got = points.read_points(str(theirs))
    assert np.array_equal(got.x3, pc.x3) and np.array_equal(got.a_im, pc.a_im)


def test_csv_format_matches_reference_reader(ref, tmp_path):
    f = tmp_path / "p.csv"
    f.write_text("x,y,z,re,im\n0.5,1,-2.5e-1,1e-3,7\n\n1 , 2 ,3,4,5\n-1,-2,-3,-4,-5e2\n")
    got = points.read_points(str(f))
    want = ref.read_points(f)
    for g, w in zip((got.x1, got.x2, got.x3, got.a_re, got.a_im), want):
        assert np.array_equal(g, w)
    assert got.size() == 3


def test_format_errors_mirror_reference(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2,3,4,5\nnot,a,number,at,all\n")
    with pytest.raises(RuntimeError, match="bad CSV line"):
        points.read_points(str(bad))
    empty = tmp_path / "empty.csv"
    empty.write_text("header only\n")
    with pytest.raises(RuntimeError, match="empty CSV point file"):
        points.read_points(str(empty))
    trunc = tmp_path / "t.ifgf"
    trunc.write_bytes(b"IFGF" + (1).to_bytes(4, "little") + (10).to_bytes(8, "little") + b"\0" * 40)
    with pytest.raises(RuntimeError, match="truncated"):
        points.read_points(str(trunc))
    ver = tmp_path / "v.ifgf"
    ver.write_bytes(b"IFGF" + (2).to_bytes(4, "little") + (0).to_bytes(8, "little"))
    with pytest.raises(RuntimeError, match="unsupported point file version"):
        points.read_points(str(ver))
    with pytest.raises(RuntimeError, match="cannot open"):
        points.read_points(str(tmp_path / "missing"))


def test_diameter_rules():
    pc = points.generate_surface(0, 1.0, 4, 1)  # 96 points: exact pairwise
    assert abs(points.diameter(pc) - 2.0) < 0.1
    big = points.generate_surface(0, 1.0, 50, 1)  # 15,000 points: box diagonal
    ex = big.x1.max() - big.x1.min()
    assert abs(points.diameter(big) - np.sqrt(3) * ex) < 1e-12


def test_cli_case_building_follows_reference():
    ap_args = ["run", "--n", "20000", "--size-lambda", "4", "--seed", "7"]
    import argparse
    p = argparse.ArgumentParser()
    sub = p.add_subparsers(dest="cmd")
    cli.add_common(sub.add_parser("run"))
    o = p.parse_args(ap_args)
    b = cli.build_case(o)
    # acceptance.cpp sphere_case(20000, 7): npd = lround(sqrt(20000/6)) = 58
    assert b.pc.size() == 6 * 58 * 58
    assert abs(b.cfg.wavenumber - 2 * np.pi * 4 / 2.0) < 1e-15
    o.kernel = "laplace"
    b = cli.build_case(o)
    assert b.cfg.wavenumber == 0.0 and not b.pc.a_im.any()
    o.kernel, o.size_lambda = "helmholtz", 0.0
    with pytest.raises(cli.ValidationError):
        cli.build_case(o)
    o.size_lambda, o.p = 4.0, [3, 5]
    with pytest.raises(cli.ValidationError):
        cli.build_case(o)


def test_cli_errors_exit_2(capsys, ifgf):
    if ifgf.device_ok():
        pytest.skip("a device is visible (the GPU test runs the CLI)")
    rc = cli.main(["run", "--n", "600"])
    assert rc == 2
    assert "error:" in capsys.readouterr().err
