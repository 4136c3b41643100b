"""CPU: the C-ABI library builds, loads, exports every symbol include/sk_b200.h
declares, fails loudly without a GPU, and the host-side mirror behaves like
the reference's host code (config parsing, grid arithmetic, error types)."""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2408_11235_b200 import build as B
    from paper_2408_11235_b200 import _native

    B.build()
    return _native


def test_library_exports_every_header_symbol(lib):
    syms = lib.header_symbols()
    assert len(syms) >= 40
    so = C.CDLL(lib.LIB)
    missing = [s for s in syms if not hasattr(so, s)]
    assert not missing, missing
    # the ctypes binding covers the whole header
    assert sorted(lib.SIGNATURES) == syms


def test_sm100a_cubin_only(lib):
    """the .so carries sm_100a SASS (and no other arch)"""
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB], capture_output=True, text=True)
    archs = {l.split(".")[-2] for l in out.stdout.split() if l.endswith(".cubin")}
    assert archs == {"sm_100a"}, out.stdout[:500]


def test_sass_uses_bulk_copies(lib):
    """the x sweep is TMA/bulk-copy driven (UBLKCP) and the v sweep uses LDGSTS"""
    sass = subprocess.run(["cuobjdump", "-sass", lib.LIB], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass
    assert "LDGSTS" in sass


def test_no_gpu_fails_loudly(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = lib.lib()
    h = C.c_void_p()
    left = (C.c_double * 1)(-1.0)
    cells = (C.c_int * 1)(8)
    dx = (C.c_double * 1)(0.25)
    rc = L.sk_ctx_create(0, 2, 1, left, cells, dx, 10.0, C.byref(h))
    assert rc == lib.SK_ERR_CUDA
    assert b"no CPU fallback" in L.sk_last_error()


def test_three_block_grid_arithmetic(lib):
    """sk_grid_three_block == Grid1D::three_block (grid.cpp:36-46), bitwise"""
    import paper_2408_11235_b200 as sk

    for nf, nc, m in [(32, 64, 1), (128, 256, 8), (512, 1024, 1), (7, 13, 3)]:
        g = sk.Grid1D.three_block(-200.0, 200.0, nf, nc, m)
        dxf = 400.0 / (2.0 * nf + float(m) * nc)
        dxc = m * dxf
        assert g.dx == [dxf, dxc, dxf]
        assert g.left == [-200.0, -200.0 + nf * dxf, (-200.0 + nf * dxf) + nc * dxc]
        assert g.cells == [nf, nc, nf]


def test_limiter_parse_mirrors_reference(sk):
    for mode in sk.LimiterConfig.MODES:
        assert sk.LimiterConfig.parse(mode).mode_string() == mode
    for bad, msg in [("weno", "unknown limiter mode"), ("foo+simple", "unknown limiter indicator"),
                     ("minmod+bar", "unknown limiter modifier")]:
        with pytest.raises(RuntimeError, match=msg):
            sk.LimiterConfig.parse(bad)
    with pytest.raises(RuntimeError, match="mass ratio"):
        sk.SpeciesParams.ion(0.0)


def test_named_configs(sk):
    c1, c3, c5 = sk.named_config("C1"), sk.named_config("C3"), sk.named_config("C5")
    assert (c1.nx, c1.v_cells, c1.k) == (128, 128, 2)
    assert (c3.nx, c3.v_cells, c3.k, c3.mu) == (2048, 4096, 3, 1836.0)
    assert c3.dof_total == 268435456
    assert c5.dof_total == 2 * (16384 * 4) ** 2
    assert sk.named_config("C2").refinement_ratio == 8


def test_cpp_mirror_compiles_and_links(lib):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    out = "/tmp/sk_test_cpp_api"
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-o", out,
           os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"),
           os.path.join(ROOT, "oracle", "_build", "libsk_oracle.so"), lib.LIB,
           "-Wl,-rpath," + os.path.dirname(lib.LIB) + ":" + os.path.join(ROOT, "oracle", "_build")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_bench_reference_arm_contract():
    """bench.py --impl reference prints one JSON line with the reference's rate"""
    import json
    import sys

    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "C1", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "DoF/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
