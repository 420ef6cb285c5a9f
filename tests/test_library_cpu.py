"""CPU-side checks of the product library: it builds for sm_100a, loads, and exports every
symbol include/llmpilot.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "llmpilot.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(llmpilot_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2410_02425_b200 import build
    return build.build()


def test_header_declares_the_survey_entry_points():
    names = _declared()
    for fn in ("llmpilot_bin", "llmpilot_fit", "llmpilot_predict", "llmpilot_recommend",
               "llmpilot_cv_leave_one_llm_out", "llmpilot_last_error", "llmpilot_ctx_create"):
        assert fn in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (llmpilot_\w+)", out))
    assert set(_declared()) <= exported


def test_library_is_sm100a_and_uses_no_fma_contraction_flag(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_strings_without_gpu(libpath):
    import paper_2410_02425_b200 as lp
    assert "sm_100a" in lp.version()
    assert lp.lib().llmpilot_last_error() == b""
    names = lp.kernel_class_names()
    assert names[5] == "hist_root" and names[7] == "hist_level"


def test_ctx_create_fails_loudly_without_gpu(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2410_02425_b200 as lp
    with pytest.raises(lp.LLMPilotError):
        lp.Context(0)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2410_02425_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "llmpilot_oracle" not in txt, f
