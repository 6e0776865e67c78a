"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a,
loads, and exports every symbol include/speedrec.h declares.  No compute
calls (there is no GPU here)."""
import ctypes as ct
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "speedrec.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sr_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1910_07776_b200.build import build_library
    return build_library()


def test_header_declares_expected_api():
    from paper_1910_07776_b200.speedrec import EXPORTS
    assert _declared() == sorted(EXPORTS)


def test_library_exports_every_declared_symbol(libpath):
    lib = ct.CDLL(libpath)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sr_[a-z_]+)$", out, flags=re.M))
    assert set(_declared()) <= exported


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath], capture_output=True,
                          text=True).stdout
    assert "DMMA.8x8x4" in sass          # the Gram contraction runs on the FP64 tensor pipe


def test_default_params_and_version(libpath):
    from paper_1910_07776_b200 import speedrec
    p = speedrec.default_params()
    assert (p.max_count, p.refine_steps, p.ridge, p.threshold, p.clamp_floor) == (3, 2, 1e-8, 1.05, 0.01)
    assert (p.learner, p.k_nn, p.top_k) == (0, 10, 64)
    assert speedrec.lib().sr_version().startswith(b"speedrec")


def test_null_context_is_an_error_not_a_crash(libpath):
    from paper_1910_07776_b200 import speedrec
    L = speedrec.lib()
    assert L.sr_evaluate(None, None, 0, 0, None) == speedrec.SR_E_ARG
    assert L.sr_load_dataset(None, None) == speedrec.SR_E_ARG
    assert L.sr_last_launch_count(None) == speedrec.SR_E_ARG
    L.sr_destroy(None)


def test_no_gpu_means_loud_failure(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1910_07776_b200 import Context, SpeedrecError
    with pytest.raises(SpeedrecError):
        Context(0)


def test_product_path_does_not_touch_oracle():
    """The CUDA path and the oracle share no code and neither imports the other."""
    pkg = os.path.join(ROOT, "paper_1910_07776_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or f == "__init__.py", f
    otxt = open(os.path.join(ROOT, "oracle", "oracle.c")).read() + open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert "paper_1910_07776_b200" not in otxt.replace("paper_1910_07776_b200/ (the CUDA path)", "").replace(
        "`paper_1910_07776_b200/`", "")


def test_learner_names_map_to_the_header_enum():
    """sr_learner values (include/speedrec.h) and their names in the binding."""
    import re
    from paper_1910_07776_b200 import SR_IBK, SR_LINREG, SR_M5P, default_params
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "speedrec.h")).read()
    enum = dict((k, int(v)) for k, v in re.findall(r"(SR_LINREG|SR_IBK|SR_M5P) = (\d+)", hdr))
    assert enum == {"SR_LINREG": SR_LINREG, "SR_IBK": SR_IBK, "SR_M5P": SR_M5P}
    assert default_params(learner="m5").learner == SR_M5P
    assert default_params(learner="ibk").learner == SR_IBK
    assert default_params().learner == SR_LINREG
    with pytest.raises(KeyError):
        default_params(learner="logistic")
