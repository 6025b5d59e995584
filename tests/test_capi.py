"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/tucomp_b200.h declares, and fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tucomp_b200.h")).read()
    return sorted(set(re.findall(r"\b(tcb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    assert "tcb_compress" in syms and "tcb_compress_device" in syms and "tcb_encode" in syms


def test_library_exports_every_declared_symbol():
    import paper_2107_01384_b200 as pkg

    lib = pkg.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(pkg.EXPORTED) <= set(declared_symbols())


def test_library_is_sm100a_only():
    import subprocess

    import paper_2107_01384_b200 as pkg

    out = subprocess.run(["cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", pkg.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # fp64 tensor-core Gram/TTM


def test_fails_loudly_without_gpu():
    import paper_2107_01384_b200 as pkg

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(pkg.TucompError, match="no CUDA device"):
        pkg.compress(pkg.SourceBuffer.from_array(np.ones((4, 4, 4))), pkg.Params(target_re=1e-2))


def test_params_struct_layout_matches_header():
    import paper_2107_01384_b200 as pkg

    # tcb_params: 17 fields incl. two 8-entry u64 arrays
    assert ctypes.sizeof(pkg._CParams) == 224
