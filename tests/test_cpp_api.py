"""The C++ drop-in header include/tucomp/pipeline.hpp (reference
pipeline.hpp:14-71 surface) compiles against libtucomp_b200.so and behaves
like the Python mirror."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = tmp_path / "cpp_api_example"
    lib = os.path.join(ROOT, "paper_2107_01384_b200")
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "cpp_api_example.cpp"), "-L", lib, "-ltucomp_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    return exe


def test_cpp_header_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by the gpu variant")
    except ImportError:
        pass
    out = subprocess.run([str(exe)], capture_output=True, text=True).stdout
    assert "no CUDA device" in out


@pytest.mark.gpu
def test_cpp_header_matches_python_mirror(tmp_path, gpu_pkg):
    exe = _build(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True).stdout
    i = np.arange(16 ** 3)
    x = (np.sin(0.1 * i) + 0.01 * np.cos(1.7 * i)).reshape(16, 16, 16)
    res = gpu_pkg.compress(gpu_pkg.SourceBuffer.from_array(x), gpu_pkg.Params(target_re=1e-2))
    assert out.strip() == f"bytes {len(res.container)}"
