"""`quake_apply` (tools/quake_apply.cpp): the reference CLI's `apply` subcommand
on the GPU path (reference tools/quake_cli.cpp:246-296, exit codes :40-42,
buffer formats core/src/io.cpp:45-111; tests mirrored: tests/test_cli.cpp:73-155)."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import CONTINUITY, EXACT, MINIMAX, QUAKE, QUAKE2
from tests.helpers import assert_bitexact, max_rel, max_ulp, restatement

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_2412_00408_b200", "bin", "quake_apply")
LOG2E = np.float32(1.4426950408889634)


def write_raw(path, x):
    x = np.ascontiguousarray(x, dtype="<f4")
    with open(path, "wb") as f:
        f.write(b"QAKE" + np.uint32(x.size).astype("<u4").tobytes() + x.tobytes())


def read_raw(path):
    b = open(path, "rb").read()
    assert b[:4] == b"QAKE"
    n = int(np.frombuffer(b[4:8], "<u4")[0])
    assert len(b) == 8 + 4 * n
    return np.frombuffer(b[8:], "<f4").copy()


def write_csv(path, x):
    with open(path, "w") as f:
        f.write("\n".join("%.9g" % v for v in np.asarray(x, np.float32)) + "\n")


def read_csv(path):
    txt = open(path).read().replace(",", " ").split()
    return np.array([np.float32(t) for t in txt], np.float32)


def run(*args):
    return subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=300)


@pytest.fixture(scope="module", autouse=True)
def _tool():
    if not os.path.exists(TOOL):
        pytest.skip("quake_apply not built")


def test_usage_and_io_exit_codes(tmp_path):
    assert run("--op", "softmax").returncode == 2                  # missing --input/--output
    assert run("--op", "foo", "--input", "a", "--output", "b").returncode == 3  # input read first
    assert run("--op", "gelu", "--input", "a", "--output", "b", "--format", "bin").returncode == 2
    assert run("--op", "gelu", "--input", "a", "--output", "b", "--kernel", "x").returncode == 2
    assert run("--op", "gelu", "--input", "a", "--output", "b", "--bias", "x").returncode == 2
    r = run("--op", "gelu", "--input", str(tmp_path / "missing.csv"), "--output", "b")
    assert r.returncode == 3 and "cannot open for reading" in r.stderr
    bad = tmp_path / "bad.raw"
    bad.write_bytes(b"NOPE\x01\x00\x00\x00\x00\x00\x80\x3f")
    r = run("--op", "exp", "--format", "raw", "--input", str(bad), "--output", str(tmp_path / "o"))
    assert r.returncode == 2 and "not a QAKE raw buffer" in r.stderr
    short = tmp_path / "short.raw"
    short.write_bytes(b"QAKE\x02\x00\x00\x00\x00\x00\x80\x3f")
    r = run("--op", "exp", "--format", "raw", "--input", str(short), "--output", str(tmp_path / "o"))
    assert r.returncode == 2 and "length mismatch" in r.stderr
    tok = tmp_path / "tok.csv"
    tok.write_text("1.0, 2.0x, 3\n")
    r = run("--op", "exp", "--input", str(tok), "--output", str(tmp_path / "o"))
    assert r.returncode == 2 and "bad numeric token" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["raw", "csv"])
def test_apply_elementwise_matches_reference(tmp_path, fmt):
    R = restatement()
    x = np.random.default_rng(3).uniform(-90, 90, 5003).astype(np.float32)
    inp, out = tmp_path / f"in.{fmt}", tmp_path / f"out.{fmt}"
    (write_raw if fmt == "raw" else write_csv)(inp, x)
    rd = read_raw if fmt == "raw" else read_csv
    x = rd(inp)  # what the tool actually parsed
    cases = [("logistic", "quake", None, R.logistic_buffer(x, QUAKE)),
             ("logistic", "quake2", "on", R.logistic_buffer(x, QUAKE2, 1)),
             ("gelu", "quake2", None, R.gelu_buffer(x, QUAKE2)),
             ("gelu", "quake", "off", R.gelu_buffer(x, QUAKE, 0))]
    c = R.coeffs_for(LOG2E, 0.0, 1)
    cases.append(("exp", "quake", None, R.quake_buffer(x, *c, *R.clamp_for(*c))))
    c2 = R.coeffs_for(LOG2E, 0.0, 0)
    cases.append(("exp", "quake2", None, R.quake2_buffer(x, *c2, CONTINUITY, *R.clamp_for(*c2))))
    for op, kern, bias, want in cases:
        args = ["apply", "--op", op, "--kernel", kern, "--format", fmt, "--input", str(inp),
                "--output", str(out)]
        if bias:
            args += ["--bias", bias]
        r = run(*args)
        assert r.returncode == 0, r.stderr
        assert_bitexact(rd(out), want, f"{op} {kern} {fmt}")
    r = run("--op", "exp", "--kernel", "quake2", "--coeffs", "minimax", "--format", fmt,
            "--input", str(inp), "--output", str(out))
    assert r.returncode == 0
    assert_bitexact(rd(out), R.quake2_buffer(x, *c2, MINIMAX, *R.clamp_for(*c2)), "minimax")
    r = run("--op", "exp", "--kernel", "exact", "--format", fmt, "--input", str(inp),
            "--output", str(out))
    assert r.returncode == 0
    small = np.abs(x) < 80
    assert max_ulp(rd(out)[small], np.exp(x[small].astype(np.float64)).astype(np.float32)) <= 2


@pytest.mark.gpu
def test_apply_softmax_rows_and_errors(tmp_path):
    R = restatement()
    cols = 256
    x = (np.random.default_rng(4).standard_normal(33 * cols) * 3).astype(np.float32)
    inp, out = tmp_path / "in.raw", tmp_path / "out.raw"
    write_raw(inp, x)
    for kern, kid in (("quake", QUAKE), ("quake2", QUAKE2)):
        r = run("--op", "softmax", "--cols", str(cols), "--kernel", kern, "--temperature", "0.5",
                "--format", "raw", "--input", str(inp), "--output", str(out))
        assert r.returncode == 0, r.stderr
        assert max_rel(read_raw(out), R.softmax_rows(x, cols, 0.5, kid)) <= 2e-6
    # --cols 0: one row spanning the buffer
    r = run("--op", "softmax", "--kernel", "quake2", "--format", "raw", "--input", str(inp),
            "--output", str(out))
    assert r.returncode == 0
    assert max_rel(read_raw(out), R.softmax_rows(x, x.size, 1.0, QUAKE2, sum_mode=1)) <= 2e-6
    # reference error behaviour: non-divisible cols, non-finite input -> exit 2, no output
    r = run("--op", "softmax", "--cols", "7", "--format", "raw", "--input", str(inp),
            "--output", str(tmp_path / "o1.raw"))
    assert r.returncode == 2 and "not divisible" in r.stderr
    xb = x.copy()
    xb[100] = np.nan
    write_raw(inp, xb)
    r = run("--op", "softmax", "--cols", str(cols), "--format", "raw", "--input", str(inp),
            "--output", str(tmp_path / "o2.raw"))
    assert r.returncode == 2 and "non-finite" in r.stderr
    assert not (tmp_path / "o2.raw").exists()


# ---- the reference's CLI cases (tests/test_cli.cpp:73-229) on quake_apply ----

@pytest.mark.gpu
def test_reference_cli_cases(tmp_path):
    inp, out = tmp_path / "in.csv", tmp_path / "out.csv"
    # apply softmax to a uniform row (test_cli.cpp:73-83)
    inp.write_text("0\n0\n0\n0\n")
    assert run("apply", "--op", "softmax", "--input", str(inp), "--output", str(out)).returncode == 0
    assert list(read_csv(out)) == [0.25] * 4
    # apply gelu maps zero to zero (:85-94)
    inp.write_text("0\n")
    assert run("apply", "--op", "gelu", "--input", str(inp), "--output", str(out)).returncode == 0
    assert list(read_csv(out)) == [0.0]
    # apply exp with the biased first-order kernel (:96-107)
    inp.write_text("1.0\n")
    assert run("apply", "--op", "exp", "--kernel", "quake", "--bias", "on", "--input", str(inp),
               "--output", str(out)).returncode == 0
    y = read_csv(out)
    assert y.size == 1 and abs(y[0] - np.e) / np.e <= 0.043
    # csv reader accepts commas and newlines (test_io.cpp:77-86)
    inp.write_text("1.5, 2.5\n3.5,\n4.5\n")
    assert run("apply", "--op", "exp", "--kernel", "exact", "--input", str(inp),
               "--output", str(out)).returncode == 0
    assert read_csv(out).size == 4
    # exact softmax through apply is stable under reapplication (:211-229)
    inp.write_text("0.25\n0.25\n0.25\n0.25\n")
    once, twice = tmp_path / "once.csv", tmp_path / "twice.csv"
    assert run("apply", "--op", "softmax", "--kernel", "exact", "--input", str(inp),
               "--output", str(once)).returncode == 0
    assert run("apply", "--op", "softmax", "--kernel", "exact", "--input", str(once),
               "--output", str(twice)).returncode == 0
    a, b = read_csv(once), read_csv(twice)
    assert np.all(np.abs(a - b) <= 2 * np.spacing(a))


def test_reference_cli_validation(tmp_path):
    """test_cli.cpp:109-123: shape, missing file, junk token, unknown op."""
    inp = tmp_path / "in.csv"
    inp.write_text("1\n2\n3\n")
    assert run("apply", "--op", "softmax", "--cols", "2", "--input", str(inp), "--output",
               str(tmp_path / "o.csv")).returncode == 2
    assert run("apply", "--op", "exp", "--input", str(tmp_path / "missing.csv"), "--output",
               str(tmp_path / "o.csv")).returncode == 3
    inp.write_text("1, banana\n")
    assert run("apply", "--op", "exp", "--input", str(inp), "--output",
               str(tmp_path / "o.csv")).returncode == 2
    assert run("apply", "--op", "transmogrify", "--input", str(inp), "--output", "x").returncode == 2


def test_apply_edge_order_follows_the_reference(tmp_path):
    """quake_cli.cpp:259-296: format, kernel and bias are parsed, then the input
    is read, then the op dispatched; --coeffs is parsed only by softmax and
    exp/QuAKE2. So an unknown op reports the missing input first (exit 3)."""
    inp = tmp_path / "in.csv"
    inp.write_text("0.5\n-1\n")
    missing = str(tmp_path / "missing.csv")
    assert run("--op", "transmogrify", "--input", missing, "--output", "x").returncode == 3
    assert run("--op", "transmogrify", "--input", str(inp), "--output", "x").returncode == 2
    assert run("--op", "gelu", "--coeffs", "bogus", "--input", missing, "--output", "x").returncode == 3
    assert run("--op", "softmax", "--coeffs", "bogus", "--input", missing,
               "--output", "x").returncode == 3
    assert run("--op", "softmax", "--coeffs", "bogus", "--input", str(inp),
               "--output", "x").returncode == 2


@pytest.mark.gpu
def test_apply_ignores_coeffs_where_the_reference_does(tmp_path):
    inp, out = tmp_path / "in.csv", tmp_path / "out.csv"
    inp.write_text("0.5\n-1\n")
    for op, kern in (("gelu", "quake2"), ("logistic", "quake2"), ("exp", "quake"), ("exp", "exact")):
        r = run("--op", op, "--kernel", kern, "--coeffs", "bogus", "--input", str(inp),
                "--output", str(out))
        assert r.returncode == 0, (op, kern, r.stderr)
    r = run("--op", "exp", "--kernel", "quake2", "--coeffs", "bogus", "--input", str(inp),
            "--output", str(out))
    assert r.returncode == 2


@pytest.mark.gpu
def test_raw_round_trip_is_deterministic(tmp_path):
    """test_cli.cpp:175-209: two runs (and a different device list) give identical bytes."""
    x = np.random.default_rng(97).uniform(-5, 5, 257).astype(np.float32)
    inp = tmp_path / "in.qak"
    write_raw(inp, x)
    outs = []
    for i, extra in enumerate(([], [], ["--devices", "0"])):
        o = tmp_path / f"o{i}.qak"
        r = run("apply", "--op", "logistic", "--kernel", "quake2", "--format", "raw",
                "--input", str(inp), "--output", str(o), *extra)
        assert r.returncode == 0, r.stderr
        outs.append(o.read_bytes())
    assert outs[0] == outs[1] == outs[2]
    assert_bitexact(read_raw(tmp_path / "o0.qak"), restatement().logistic_buffer(x, QUAKE2))
