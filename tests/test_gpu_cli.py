"""The `tucomp` CLI on the device: CLI-vs-API byte equality of the container
(SPEC.md's CLI parity requirement), decompress output equal to
pipeline::decompress, the measured error against the oracle's decoder, and the
sweep CSV (reference tools/tucomp_main.cpp:172-272)."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2107_01384_b200", "tucomp")


def run(*args):
    r = subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r.stdout


def _machine(out):
    return {l.split()[0][7:]: float(l.split()[1]) for l in out.splitlines() if l.startswith("report.")}


def test_compress_is_deterministic(gpu_pkg):
    x = synth.small("sin_decay", (40, 32, 24), seed=7)
    a = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-4)).container
    b = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-4)).container
    assert a == b


@pytest.mark.parametrize("dtype,flags,params", [
    (np.float64, [], dict(target_re=1e-4)),
    (np.float32, ["--coder", "rans", "--vectorization", "zorder"], dict(target_re=1e-3, coder=1, method=2)),
    (np.uint16, ["--storage-order", "3,1,2", "--block-size", "1024", "--no-split-planes"],
     dict(target_re=1e-3, storage_order=(2, 0, 1), block_size=1024, split_planes=False)),
    (np.int16, ["--simple-factor-weights", "--vectorization", "zigzag", "--rtmss", "0.3"],
     dict(target_re=1e-3, simple_factor_weights=True, method=1, rtmss=0.3)),
    (np.float32, ["--mode-order", "2,3,1"], dict(target_re=1e-3, mode_order=(1, 2, 0))),
])
def test_cli_compress_matches_api(tmp_path, gpu_pkg, dtype, flags, params):
    shape = (36, 28, 20)
    base = synth.small("blobs", shape, seed=8)
    if np.issubdtype(dtype, np.integer):
        x = np.round((base - base.min()) / np.ptp(base) * 3000).astype(dtype)
    else:
        x = base.astype(dtype)
    skip = 16
    raw = tmp_path / "in.raw"
    raw.write_bytes(b"\x00" * skip + x.tobytes())
    out = tmp_path / "c.tkc"
    text = run("compress", "-i", raw, "--shape", ",".join(map(str, shape)), "--dtype", np.dtype(dtype).name,
               "--skip-bytes", skip, "-o", out, "--machine",
               *(["--target-re", params["target_re"]] if "target_re" in params else []), *flags)
    prm = gpu_pkg.Params(**params)
    api = gpu_pkg.compress(gpu_pkg.SourceBuffer(b"\x00" * skip + x.tobytes(), gpu_pkg.Dtype(oracle.DTYPES[np.dtype(dtype)]),
                                                list(shape), skip), prm)
    cont = out.read_bytes()
    assert cont == api.container  # CLI-vs-API byte equality
    m = _machine(text)
    assert m["bytes"] == len(cont)
    # measured error: device ingest + decompress + SSE vs the oracle's decoder in numpy
    y = oracle.decompress(cont, shape)
    xd = x.astype(np.float64)
    sse = float(((y - xd) ** 2).sum())
    # report lines print 6 significant digits
    tol = 1e-5
    assert abs(m["achieved_sse"] - sse) <= tol * sse + 1e-300
    assert m["achieved_re"] <= params["target_re"] * 1.05
    assert abs(m["estimate_sse"] - api.estimate.total()) <= 1e-5 * api.estimate.total()
    # decompress through the CLI == pipeline::decompress
    rec = tmp_path / "out.raw"
    text = run("decompress", "-i", out, "-o", rec)
    assert text.startswith(f"wrote {x.nbytes} bytes ({np.dtype(dtype).name}, shape {' '.join(map(str, shape))})")
    assert rec.read_bytes() == gpu_pkg.decompress(cont).bytes


def test_cli_internal_float32_fails_like_api(tmp_path, gpu_pkg):
    """internal_float32 throws in factorize exactly where the reference throws
    (DESIGN.md §0); the CLI reports the same text with exit code 1."""
    x = synth.small("sin", (20, 16, 12), seed=2).astype(np.float32)
    raw = tmp_path / "in.raw"
    raw.write_bytes(x.tobytes())
    with pytest.raises(gpu_pkg.TucompError) as ei:
        gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-3, internal_float32=True))
    r = subprocess.run([EXE, "compress", "-i", raw, "--shape", "20,16,12", "--dtype", "float32", "-o",
                        tmp_path / "c.tkc", "--target-re", "1e-3", "--internal-float32"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 1 and r.stderr.strip() == f"error: {ei.value}"


def test_cli_no_verify_and_target_sse(tmp_path, gpu_pkg):
    x = synth.small("sin", (24, 24, 24), seed=3)
    raw = tmp_path / "in.raw"
    raw.write_bytes(x.tobytes())
    out = tmp_path / "c.tkc"
    text = run("compress", "-i", raw, "--shape", "24,24,24", "-o", out, "--target-sse", "1e-2", "--machine",
               "--no-verify")
    m = _machine(text)
    assert m["achieved_sse"] == 0 and m["achieved_re"] == 0  # no measurement pass (tucomp_main.cpp:177)
    api = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_sse=1e-2))
    assert out.read_bytes() == api.container


def test_cli_sweep_csv(tmp_path, gpu_pkg):
    x = synth.small("sin_decay", (32, 24, 20), seed=9)
    raw = tmp_path / "in.raw"
    raw.write_bytes(x.tobytes())
    csv = tmp_path / "s.csv"
    run("sweep", "-i", raw, "--shape", "32,24,20", "--target-re-grid", "1e-2,1e-3,1e-4", "--rtmss-grid", "0.5,0.8",
        "-o", csv)
    lines = csv.read_text().splitlines()
    assert lines[0] == "target_re,achieved_re,factor,rtmss,comp_ms,decomp_ms"
    rows = [list(map(float, l.split(","))) for l in lines[1:]]
    assert len(rows) == 6
    assert [r[3] for r in rows] == [0.5] * 3 + [0.8] * 3
    for t, a, f, _, c, d in rows:
        assert 0 < a <= 1.05 * t and f > 1 and c > 0 and d > 0
    # stdout form with a failing cell (lossless target rejected per cell, tucomp_main.cpp:262-267)
    r = subprocess.run([EXE, "sweep", "-i", raw, "--shape", "32,24,20", "--target-re-grid", "0,1e-2"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0
    out = r.stdout.splitlines()
    assert out[1] == "0,nan,nan,0.5,nan,nan" and "sweep cell re=0 rtmss=0.5 failed" in r.stderr
    assert float(out[2].split(",")[1]) <= 1.05e-2
