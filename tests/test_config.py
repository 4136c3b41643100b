"""CPU: the run-configuration surface against the reference.

The reference's RunConfig (config.cpp, compiled in place into oracle/_ref) is
the oracle; both mirrors -- Python ``RunConfig`` and the C++
``include/solkin_b200_config.hpp`` -- must produce the same echo, violations,
nsteps and error messages for the same presets / files / key=value overrides.
``sk_shift_matrices`` (the `solkin matrices` table) must equal the reference's
``build_shift_matrices`` bitwise. None of this needs a GPU.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = "/tmp/sk_config_tool"

PRESETS = ["", "blob-desk", "injection-desk", "blob-paper", "injection-paper", "nope"]

# (key, value) overrides applied verbatim through apply_kv
KV_CASES = [
    [],
    [("L", "100"), ("dt", "0.05"), ("k", "2"), ("mu", "1836"), ("t_final", "1.25")],
    [("sigma", "3.5"), ("t0", "1e3"), ("vmax_e", "+8"), ("vmax_i", ".5")],
    [("mesh.fine_block_cells", "128"), ("mesh.coarse_block_cells", "256"),
     ("mesh.refinement_ratio", "8"), ("v_cells", "512")],
    [("limiter", "minmod+line"), ("limiter.threshold", "0.25"), ("adaptivity.v_adjust", "off"),
     ("adaptivity.p", "0.1"), ("adaptivity.gamma", "0"), ("adaptivity.tol", "1e-12")],
    [("poisson.penalty_scale", "20"), ("output.dir", "run a"), ("output.cadence", "5"),
     ("output.snapshot_cadence", "100"), ("output.profile_cadence", "50"), ("threads", "8")],
    [("scenario", "injection"), ("adaptivity.v_adjust", "true"), ("adaptivity.v_adjust", "0")],
    # hex / special floats / leading whitespace: what std::stod accepts
    [("L", "0x1p4"), ("dt", " 0.2"), ("t_final", "inf"), ("mu", "nan")],
    [("sigma", "-nan"), ("t0", "1e-5")],
    # violations (all of them)
    [("scenario", "x"), ("L", "0"), ("dt", "-1"), ("k", "7"), ("mu", "0"), ("t_final", "-1"),
     ("t0", "0"), ("vmax_e", "0"), ("vmax_i", "-2"), ("mesh.fine_block_cells", "0"),
     ("mesh.coarse_block_cells", "-1"), ("mesh.refinement_ratio", "0"), ("v_cells", "0"),
     ("limiter", "minmod+"), ("limiter.threshold", "0"), ("adaptivity.p", "0.5"),
     ("adaptivity.gamma", "0.5"), ("adaptivity.tol", "0"), ("poisson.penalty_scale", "0"),
     ("output.cadence", "0"), ("output.snapshot_cadence", "-1"), ("output.profile_cadence", "-3"),
     ("threads", "0")],
    [("k", "-1"), ("adaptivity.gamma", "-0.1")],
    # parse errors (the first bad key throws)
    [("L", "12abc")],
    [("L", "")],
    [("dt", "1e400")],
    [("t0", "1e-320")],
    [("k", "3.0")],
    [("k", "0x10")],
    [("k", "2147483648")],
    [("k", " 4")],
    [("k", "4 ")],
    [("adaptivity.v_adjust", "yes")],
    [("nosuch", "1")],
    [("mesh.cells", "4")],
]

# nsteps = lround(t_final / dt): exact halves round away from zero
NSTEP_CASES = [("1", "0.1"), ("0.25", "0.1"), ("0.35", "0.1"), ("2.5", "1"), ("3.5", "1"),
               ("0", "0.1"), ("8000", "0.1"), ("0.15", "0.1")]

CONFIG_FILE = """# a config file with comments, blank lines and odd spacing
scenario = injection   # trailing comment
  L=150
dt\t=\t0.05\r
mesh.fine_block_cells = 64

limiter = sldg
output.dir = my out # the value is trimmed, inner spaces kept
# key = commented out
"""


@pytest.fixture(scope="module")
def sk():
    import paper_2408_11235_b200 as sk

    return sk


def py_eval(sk, preset="", file="", kv=(), resolve=False):
    try:
        c = sk.RunConfig.preset(preset) if preset else sk.RunConfig()
        if file:
            c.apply_file(file)
        for k, v in kv:
            c.apply_kv(k, v)
        if resolve:
            c.resolve()
        return ("ok", c.echo(), c.violations(), c.nsteps())
    except RuntimeError as e:
        return ("error", str(e))


@pytest.fixture(scope="module")
def tool():
    if not shutil.which("g++"):
        pytest.skip("no g++")
    from paper_2408_11235_b200 import _native

    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-o", TOOL,
           os.path.join(ROOT, "tests", "cpp", "config_tool.cpp"), _native.LIB,
           "-Wl,-rpath," + os.path.dirname(_native.LIB)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return TOOL


def cpp_run(tool, *args):
    r = subprocess.run([tool, *args], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    head, _, rest = r.stdout.partition("\n")
    if head == "error":
        return ("error", rest)
    echo, viol, n = rest.split("--\n")
    return ("ok", echo, [x for x in viol.split("\n") if x], int(n))


def cpp_eval(tool, preset="", file="", kv=(), resolve=False):
    args = ["eval", preset or "-", file or "-", "1" if resolve else "0"]
    for k, v in kv:
        args += [k, v]
    return cpp_run(tool, *args)


@pytest.mark.parametrize("preset", PRESETS)
@pytest.mark.parametrize("resolve", [False, True])
def test_presets_match_reference(ref, sk, tool, preset, resolve):
    want = ref.config_eval(preset=preset, resolve=resolve)
    assert py_eval(sk, preset, resolve=resolve) == want
    assert cpp_eval(tool, preset, resolve=resolve) == want


@pytest.mark.parametrize("case", range(len(KV_CASES)))
def test_key_value_overrides_match_reference(ref, sk, tool, case):
    kv = KV_CASES[case]
    for resolve in (False, True):
        want = ref.config_eval(kv=kv, resolve=resolve)
        assert py_eval(sk, kv=kv, resolve=resolve) == want, kv
        assert cpp_eval(tool, kv=kv, resolve=resolve) == want, kv


def test_nsteps_rounding_matches_reference(ref, sk, tool):
    for t, dt in NSTEP_CASES:
        kv = [("t_final", t), ("dt", dt)]
        want = ref.config_eval(kv=kv)
        assert want[0] == "ok"
        assert py_eval(sk, kv=kv)[3] == want[3], (t, dt)
        assert cpp_eval(tool, kv=kv)[3] == want[3], (t, dt)


def test_config_file_matches_reference(ref, sk, tool, tmp_path):
    good = tmp_path / "good.cfg"
    good.write_text(CONFIG_FILE)
    no_eq = tmp_path / "bad.cfg"
    no_eq.write_text("L = 3\n\njust a line\n")
    bad_num = tmp_path / "num.cfg"
    bad_num.write_text("dt = fast\n")
    unknown = tmp_path / "key.cfg"
    unknown.write_text("mesh.blocks = 3")  # no trailing newline
    missing = tmp_path / "missing.cfg"
    for path, preset in [(good, ""), (good, "blob-paper"), (no_eq, ""), (bad_num, ""),
                         (unknown, ""), (missing, "")]:
        for resolve in (False, True):
            want = ref.config_eval(preset=preset, file=str(path), resolve=resolve)
            assert py_eval(sk, preset, str(path), resolve=resolve) == want, path.name
            assert cpp_eval(tool, preset, str(path), resolve=resolve) == want, path.name
    assert ref.config_eval(file=str(good))[1].startswith("scenario = injection\nL = 150\n")


def test_echo_round_trips(sk, tmp_path):
    """echo() is re-ingestible: file(echo(c)) == c"""
    c = sk.RunConfig.preset("injection-paper")
    for k, v in KV_CASES[1] + KV_CASES[4] + KV_CASES[5]:
        c.apply_kv(k, v)
    c.resolve()
    path = tmp_path / "echo.cfg"
    path.write_text(c.echo())
    assert sk.RunConfig.from_file(str(path)) == c


def test_layered_resolution_matches_cmd_run(ref, sk, tool, tmp_path):
    """cmd_run (solkin_main.cpp:20-28): preset -> file -> --limiter/--out/--threads -> resolve -> validate"""
    good = tmp_path / "good.cfg"
    good.write_text(CONFIG_FILE)
    for preset, limiter, out, threads in [("blob-paper", "meanerr+simple", "o2", 4),
                                          ("", "", "", 0), ("injection-desk", "bogus", "", 0)]:
        kv = []
        if limiter:
            kv.append(("limiter", limiter))
        if out:
            kv.append(("output.dir", out))
        if threads > 0:
            kv.append(("threads", str(threads)))
        want = ref.config_eval(preset=preset, file=str(good), kv=kv, resolve=True)
        got = cpp_run(tool, "layered", str(good), preset or "-", limiter or "-", out or "-", str(threads))
        if want[2]:
            assert got == ("error", "invalid configuration:" + "".join("\n  " + v for v in want[2]))
        else:
            assert got == want


def test_to_c_carries_the_step_keys(sk):
    c = sk.RunConfig.preset("injection-paper")
    c.apply_kv("limiter", "meanerr+line")
    c.apply_kv("limiter.threshold", "0.7")
    c.resolve()
    cc = c.to_c()
    assert (cc.scenario, cc.refinement_ratio, cc.v_cells, cc.fine_block_cells) == (1, 8, 150, 100)
    assert (cc.limiter.indicator, cc.limiter.modifier, cc.limiter.threshold) == (2, 2, 0.7)
    assert cc.sigma == 0.1 * 200.0


@pytest.mark.parametrize("k", range(7))
def test_shift_matrices_bitwise(ref, sk, k):
    """sk_shift_matrices == build_shift_matrices (advection.cpp:27-66), bitwise, from the C ABI"""
    for alpha in (0.0, 1e-12, 0.125, 1.0 / 3.0, 0.5, 0.7071067811865476, 1.0 - 2.0 ** -52):
        A, B = sk.build_shift_matrices(k, alpha)
        rA, rB = ref.shift_matrices(k, alpha)
        assert np.array_equal(A.ravel(), np.asarray(rA).ravel()), (k, alpha)
        assert np.array_equal(B.ravel(), np.asarray(rB).ravel()), (k, alpha)


def test_matrices_text_matches_reference(ref, sk, tool):
    for alpha, order in [(0.0, 0), (0.3, 1), (0.25, 2), (0.6180339887498949, 3), (0.9, 6)]:
        want = ref.matrices_text(alpha, order)
        assert sk.matrices_text(alpha, order) == want
        r = subprocess.run([tool, "matrices", repr(alpha), str(order)], capture_output=True, text=True)
        assert r.stdout == want


def test_shift_matrices_errors(sk):
    with pytest.raises(RuntimeError, match=r"alpha must be in \[0,1\)"):
        sk.build_shift_matrices(3, 1.0)
    with pytest.raises(RuntimeError, match="k must be in 0..6"):
        sk.build_shift_matrices(7, 0.5)
