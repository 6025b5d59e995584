"""The `tucomp` CLI (reference proj/tools/tucomp_main.cpp:276-350) built on the
public C++ surface: argument handling, exit codes and the host-only `info`
subcommand, here without a GPU.  The device subcommands are in test_gpu_cli.py."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2107_01384_b200", "tucomp")


def run(*args):
    assert os.path.exists(EXE), "CLI not built: run __graft_entry__.build()"
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=300)


def test_usage_and_unknown_subcommand():
    r = run()
    assert r.returncode == 2 and "usage: tucomp" in r.stderr
    assert run("--help").returncode == 0
    r = run("frobnicate")
    assert r.returncode == 2 and "unknown subcommand frobnicate" in r.stderr


@pytest.mark.parametrize("args,msg", [
    (("compress", "-o", "x"), "-i is required"),
    (("compress", "-i", "a", "-o", "x"), "--shape is required"),
    (("decompress", "-i", "a"), "-o is required"),
    (("info",), "-i is required"),
    (("sweep", "-i", "a", "--shape", "2,2"), "--target-re-grid is required"),
    (("info", "-i", "a", "--bogus"), "unknown argument --bogus"),
    (("compress", "-i", "a", "--shape", "2,2", "-o", "x", "--target-re", "abc"), "bad value for --target-re"),
    (("compress", "-i", "a", "--shape", "2,2", "-o", "x", "--machine=1"), "--machine takes no value"),
])
def test_usage_errors(args, msg):
    r = run(*args)
    assert r.returncode == 2 and msg in r.stderr


@pytest.mark.parametrize("extra,msg", [
    ((), "one of --target-re / --target-sse is required"),
    (("--target-re", "1e-3", "--target-sse", "1"), "--target-re and --target-sse are mutually exclusive"),
    (("--target-re", "0"), "--target-re 0 requests lossless output"),
    (("--target-re", "1e-3", "--dtype", "float16"), "unknown dtype float16"),
    (("--target-re", "1e-3", "--coder", "huffman"), "unknown coder huffman"),
    (("--target-re", "1e-3", "--vectorization", "hilbert"), "unknown vectorization method hilbert"),
    (("--target-re", "1e-3", "--mode-order", "0,1"), "mode orders are 1-based"),
])
def test_compress_errors_before_device_work(tmp_path, extra, msg):
    """tucomp_main.cpp:77-119,338-342: flag validation throws tucomp::Error,
    printed as "error: ..." with exit code 1."""
    f = tmp_path / "in.raw"
    f.write_bytes(np.zeros(8).tobytes())
    r = run("compress", "-i", f, "--shape", "2,4", "-o", tmp_path / "o.tkc", *extra)
    assert r.returncode == 1 and r.stderr.startswith("error: ") and msg in r.stderr


def test_missing_input_file(tmp_path):
    r = run("info", "-i", tmp_path / "nope")
    assert r.returncode == 1 and "error: cannot open" in r.stderr


def _fields(text):
    out = {}
    for line in text.splitlines():
        k, _, v = line.partition(":")
        out[k.strip()] = v.strip()
    return out


@pytest.mark.parametrize("opts", [dict(), dict(coder=1, method=2, storage_order=(2, 0, 1), block_size=512),
                                  dict(split=False, simple=True, method=1)])
def test_info_on_oracle_containers(tmp_path, opts):
    """cmd_info (tucomp_main.cpp:196-228) through read_container's host parse."""
    x = synth.small("sin_decay", (24, 20, 16), seed=5).astype(np.float32)
    info = oracle.compress(x, target_re=1e-3, **opts)
    f = tmp_path / "c.tkc"
    f.write_bytes(info.container)
    r = run("info", "-i", f)
    assert r.returncode == 0, r.stderr
    v = _fields(r.stdout)
    assert v["format version"] == "1" and v["source dtype"] == "float32" and v["internal"] == "float64"
    assert v["order"] == "3" and v["mode sizes"] == "24 20 16"
    assert v["ranks"] == " ".join(map(str, info.ranks))
    import paper_2107_01384_b200 as pkg

    h = pkg.read_container(info.container)
    if "storage_order" in opts:
        assert h.storage_order == opts["storage_order"]
    assert v["storage order"] == " ".join(str(i + 1) for i in h.storage_order)
    assert v["processing order"] == " ".join(str(i + 1) for i in h.processing_order)
    assert v["block size"] == str(h.block_size) and v["scale exponent"] == str(h.core_scale_exponent)
    assert v["vectorization"] == ["lex", "zigzag", "zorder"][opts.get("method", 0)]
    assert v["entropy coder"] == ["ac", "rans"][opts.get("coder", 0)]
    assert v["split planes"] == ("no" if opts.get("split") is False else "yes")
    assert v["factor weights"] == ("slice-norm" if opts.get("simple") else "alpha")
    assert v["compressed size"] == f"{len(info.container)} bytes"
    assert v["original size"] == f"{x.nbytes} bytes"
    want = np.sqrt(h.estimate_sse / h.norm_sq)
    assert abs(float(v["recorded error"].split()[0]) - want) <= 1e-5 * want


def test_info_zero_container_and_corruption(tmp_path):
    f = tmp_path / "z.tkc"
    f.write_bytes(oracle.compress(np.zeros((4, 4, 4)), target_re=1e-3).container)
    r = run("info", "-i", f)
    assert r.returncode == 0 and "content:         constant zero" in r.stdout
    good = oracle.compress(synth.small("sin", (12, 10, 8), seed=1), target_re=1e-3).container
    f.write_bytes(good[:-5])
    r = run("info", "-i", f)
    assert r.returncode == 1 and "error: container: truncated" in r.stderr
    f.write_bytes(b"JUNK" + good[4:])
    r = run("info", "-i", f)
    assert r.returncode == 1 and r.stderr.strip() == "error: container: bad magic"
