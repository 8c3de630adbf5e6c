"""CPU-side tests of the product library (no GPU needed): the C ABI loads and
exports every entry point include/ifgf_b200.h declares, the host-only entry
points match the oracle and the reference, and compute entry points fail
loudly (no CPU fallback) when no sm_100 device is visible."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "ifgf_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ifgf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(ifgf):
    from paper_2112_15198_b200 import _lib
    names = declared_functions()
    assert len(names) >= 30
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), f"{n} declared in ifgf_b200.h but not exported"
        assert n in _lib.SIGNATURES, f"{n} not bound in _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) <= set(names)
    assert ifgf._lib.lib.ifgf_abi_version() == 2


def test_library_is_sm100a_only(ifgf):
    from paper_2112_15198_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_default_params_match_reference(ifgf):
    from paper_2112_15198_b200._lib import CParams
    p = CParams()
    ifgf._lib.lib.ifgf_default_params(ctypes.byref(p))
    # engine.hpp:12-19, interp.hpp:11-14
    assert (p.depth, p.box_lambda, p.points_per_box) == (0, 0.25, 64)
    assert (p.base_s, p.base_theta, p.base_phi) == (1, 2, 4)
    assert (p.p_s, p.p_theta, p.p_phi) == (3, 5, 5)
    e = ifgf.EngineParams()
    assert (e.box_lambda, e.points_per_box, e.orders.total()) == (0.25, 64, 75)


def test_choose_depth_through_c_abi(ifgf, oracle):
    # test_engine.cpp:371-383 KATs, and the oracle on a sweep
    p = ifgf.EngineParams()
    assert ifgf.choose_depth(100000, 16.0, 2 * math.pi, p) == 7
    assert ifgf.choose_depth(100000, 16.0 * (1 + 1e-6), 2 * math.pi, p) == 7
    assert ifgf.choose_depth(100000, 16.0, 2 * math.pi, ifgf.EngineParams(depth=5)) == 5
    assert ifgf.choose_depth(100, 1.0, 0.0, p) == 3
    assert ifgf.choose_depth(1 << 30, 1.0, 0.0, p) <= 21
    from bindings import Params
    for n in [2, 100, 5000, 98304, 1572864, 6291456, 25165824]:
        for side in [2.0000019, 1.0, 7.3]:
            for k in [0.0, 8 * math.pi, 32 * math.pi, 256 * math.pi]:
                assert ifgf.choose_depth(n, side, k, p) == oracle.choose_depth(n, side, k,
                                                                               Params())


def test_baseline_config_depths(ifgf):
    # C1 -> D=6, C2 -> D=8, C3 rule -> D=10
    for name, want in [("C1", 6), ("C2", 8), ("C3", 10)]:
        c = ifgf.configs.CONFIGS[name]
        pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
        ext = max(np.ptp(pc.x1), np.ptp(pc.x2), np.ptp(pc.x3))
        side = max((1 + 1e-6) * ext, 1e-9)
        kappa = 0.0 if c.kind == 1 else c.kappa
        assert ifgf.choose_depth(c.n, side, kappa, ifgf.EngineParams()) == want, name


def test_generator_matches_oracle_bitwise(ifgf, oracle):
    for shape, c, dens, seed in [(0, 1.0, 0, 7), (1, 0.25, 0, 8), (0, 1.0, 1, 9)]:
        a = ifgf.generate(4000, shape, c, dens, seed)
        b = oracle.generate(4000, shape, c, dens, seed)
        for u, v in zip((a.x1, a.x2, a.x3, a.a_re, a.a_im), b):
            assert np.array_equal(u, v)
    pc = ifgf.generate(20000, 1, 0.25, 0, 4)
    assert np.allclose(pc.x1 ** 2 + pc.x2 ** 2 + (pc.x3 / 0.25) ** 2, 1.0, atol=1e-14)
    assert np.all(np.abs(pc.a_re) <= 1) and np.all(np.abs(pc.a_im) <= 1)


def test_sample_indices_matches_oracle_and_reference(ifgf, oracle):
    for n, m, seed in [(10, 10, 1), (98304, 1000, 2), (1572864, 1000, 3)]:
        assert np.array_equal(ifgf.sample_indices(n, m, seed), oracle.sample_indices(n, m, seed))
    with pytest.raises(ifgf.InvalidArgument):
        ifgf.sample_indices(5, 6, 1)


def test_sample_indices_matches_reference(ifgf, ref):
    assert np.array_equal(ifgf.sample_indices(98304, 1000, 2), ref.sample_indices(98304, 1000, 2))


def test_compute_entry_points_fail_loudly_without_device(ifgf):
    if ifgf.device_ok():
        pytest.skip("a device is visible")
    pc = ifgf.generate(100, 0, 1.0, 0, 1)
    cfg = ifgf.KernelConfig(ifgf.KernelKind.Helmholtz, 3.0)
    with pytest.raises(ifgf.IFGFRuntimeError):
        ifgf.apply(pc, cfg)
    with pytest.raises(ifgf.IFGFRuntimeError):
        ifgf.Plan.from_cloud(pc, cfg)
    with pytest.raises(ifgf.IFGFRuntimeError):
        ifgf.direct_eval(pc, cfg)


def test_argument_errors_mirror_reference(ifgf):
    cfg = ifgf.KernelConfig(ifgf.KernelKind.Helmholtz, 3.0)
    one = ifgf.generate(1, 0, 1.0, 0, 1)
    with pytest.raises(ifgf.InvalidArgument):  # engine.cpp:261 need two points
        ifgf.apply(one, cfg)
    pc = ifgf.generate(10, 0, 1.0, 0, 1)
    bad = ifgf.EngineParams(orders=ifgf.InterpOrders(13, 5, 5))
    with pytest.raises(ifgf.InvalidArgument):  # engine.cpp:76-77 unsupported orders
        ifgf.Plan.from_cloud(pc, cfg, bad)


def test_reference_acceptance_runner_binds_the_gpu_library(ifgf):
    """oracle/_ref/ifgf_acceptance_b200 is the reference's acceptance.cpp
    linked through integration/ref_apply_b200.cpp: its ifgf::apply must be
    the shim's (calls into libifgf_b200.so), and without a device that call
    fails loudly with the library's message instead of running the
    reference's CPU engine."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "ifgf_acceptance_b200")
    if not os.path.exists(exe):
        pytest.skip("acceptance runner not built (needs /root/reference)")
    libs = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libifgf_b200.so" in libs
    syms = subprocess.run(["nm", exe], capture_output=True, text=True).stdout
    apply_sym = "_ZN4ifgf5applyERNS_10PointCloudERKNS_12KernelConfigERKNS_12EngineParamsE"
    kinds = {ln.split()[-2] for ln in syms.splitlines() if ln.endswith(" " + apply_sym)}
    assert kinds == {"T"}, kinds  # one strong definition: the shim
    if ifgf.device_ok():
        pytest.skip("a device is visible (tests/test_gpu_acceptance.py runs it)")
    p = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=120)
    assert p.returncode != 0 and "libifgf_b200 has no CPU path" in p.stderr, p.stderr[-500:]
