"""CPU-side checks of the C ABI library (no GPU here): it builds, loads and
exports every symbol include/bl.h declares, and compute entry points fail
loudly (BL_ERR_CUDA) instead of falling back to a CPU path."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "bl.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(bl_[a-z_0-9]+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["bl_load_design", "bl_fit_path", "bl_cv", "bl_free", "bl_lambda_max", "bl_last_error"]:
        assert s in syms


def test_library_builds_and_exports_every_declared_symbol():
    from paper_1701_05936_b200 import build
    lib_path = build.build()
    L = ctypes.CDLL(lib_path)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    from paper_1701_05936_b200 import EXPORTS
    assert sorted(EXPORTS) == declared_symbols()


def test_sass_is_sm100a_with_tensor_core_scan():
    """The int8 scan is an IMMA (s8 tensor-core) kernel; everything is sm_100a."""
    import subprocess
    from paper_1701_05936_b200 import build
    lib_path = build.build()
    out = subprocess.run(["cuobjdump", "-lelf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    sec = sass.split("Function : _ZN2bl9k_scan_i8")[1].split("Function :")[0]
    assert "IMMA.16832.S8.S8" in sec


def test_sass_batched_scan_is_tcgen05():
    """The fp32 fold-batched scan issues tcgen05 MMAs on SM pairs (UTCIMMA.2CTA) with the A operand
    written to tensor memory (STTM) and the accumulators read back from it (LDTM)."""
    import subprocess
    from paper_1701_05936_b200 import build
    sass = subprocess.run(["cuobjdump", "-sass", build.build()], capture_output=True, text=True).stdout
    sec = sass.split("Function : _ZN2bl15k_scan_batch_tcILi11EEE")[1].split("Function :")[0]
    for ins in ("UTCIMMA.2CTA", "STTM", "LDTM", "UTCBAR.2CTA.MULTICAST"):
        assert ins in sec, ins


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1701_05936_b200 import bl
    X = np.zeros((4, 8))
    with pytest.raises(bl.BLError) as e:
        bl.bl_load_design(X, 8)
    assert e.value.code == bl.BL_ERR_CUDA
    assert "no CUDA device" in str(e.value) or "CUDA" in str(e.value)


def test_argument_validation_precedes_device_use():
    from paper_1701_05936_b200 import bl
    with pytest.raises(bl.BLError) as e:
        bl.bl_load_design(np.zeros((4, 1)), 1)       # n = 1 < 2
    assert e.value.code == bl.BL_ERR_ARG
    with pytest.raises(bl.BLError) as e:
        bl.bl_load_design(np.zeros((4, 20000)), 20000)   # n > 16384
    assert e.value.code == bl.BL_ERR_ARG
