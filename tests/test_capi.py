"""C-ABI library: loads, exports every symbol include/ffca.h declares, and
fails loudly (no CPU fallback) when no B200 is visible."""
import ctypes as C
import re

import pytest

from conftest import HAS_GPU, ROOT


def header_symbols():
    text = (ROOT / "include" / "ffca.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void\*?|long long|const char\*)\s+(ffca_\w+)\s*\(", text, re.M)))


def test_header_matches_binding_exports():
    from paper_2101_08563_b200 import _lib
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(built):
    lib = C.CDLL(str(ROOT / "paper_2101_08563_b200" / "libffca.so"))
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_library_targets_sm100a(built):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          str(ROOT / "paper_2101_08563_b200" / "libffca.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(built):
    from paper_2101_08563_b200 import _lib
    with pytest.raises(_lib.CudaError):
        _lib.Context(0)


def test_invalid_arguments_rejected_before_device(built):
    from paper_2101_08563_b200 import _lib
    L = _lib.lib()
    d = _lib.Dims(1, 4, 9, 2, 10)  # dim 9 unsupported
    o = _lib.FitOpts(0, 1, 1, 0, 1, 0, 0)
    # A null context is rejected as an invalid argument, never computed on CPU.
    assert L.ffca_fit(None, d, o, None, None, None, None, None, None, None, None) == 1
