"""The C-ABI library loads and exports every symbol include/fstk_gpu.h declares
(no compute calls: this runs without a GPU)."""
import ctypes as C
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "fstk_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fstk_gpu_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_boundary():
    names = _declared()
    for must in ("fstk_gpu_evaluate_batch", "fstk_gpu_evaluate", "fstk_gpu_mode_values",
                 "fstk_gpu_reestimate_core", "fstk_gpu_sketch", "fstk_gpu_build_design_rows",
                 "fstk_gpu_mixed_matrix", "fstk_gpu_model_create", "fstk_gpu_refit_begin"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1907_05884_b200 import _lib

    L = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == _declared()
    _lib.lib()  # the binding itself resolves every symbol
    assert L.fstk_gpu_abi_version() == 3


def test_library_is_sm100a():
    """The cubin inside the library targets sm_100a (no PTX-only/other-arch build)."""
    import subprocess

    from paper_1907_05884_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        import pytest

        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_is_loud_on_cpu():
    """Without a GPU the product raises instead of falling back to the CPU."""
    import numpy as np
    import pytest

    from paper_1907_05884_b200 import _lib, synth

    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    m = synth.random_model((2, 2), (3, 3), 2, seed=0)
    with pytest.raises(Exception):
        m.evaluate_batch(np.zeros((4, 2)) + 0.5)
