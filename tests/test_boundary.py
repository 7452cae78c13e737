"""The C-ABI library loads and exports every symbol include/emoe.h declares,
and fails loudly when missing (no GPU needed)."""
import ctypes
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "emoe.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(emoe_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2503_06823_b200 import _lib

    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, f"missing exports: {missing}"
    assert set(syms) == set(_lib.EXPORTED), set(syms) ^ set(_lib.EXPORTED)


def test_library_is_sm100a():
    so = ROOT / "paper_2503_06823_b200" / "lib" / "libemoe.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout[:500]
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "tcgen05.mma missing from the FFN kernels"
    assert "UTMALDG" in sass, "TMA loads missing from the FFN kernels"
    assert "LDTM" in sass, "tcgen05.ld missing from the FFN epilogue"


def test_version_and_error_plumbing():
    from paper_2503_06823_b200 import ValidationError, _lib
    from paper_2503_06823_b200.moesim import check

    assert _lib.lib.emoe_version() == 1
    # a validation error without touching the GPU: bad layer config
    cfg = _lib.LayerConfig(512, 1024, 0, 2, 0, 0, 0, 4, 128, 0)
    h = ctypes.c_void_p()
    rc = _lib.lib.emoe_layer_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc == 2
    assert b"num_experts" in _lib.lib.emoe_last_error()
    try:
        check(rc)
    except ValidationError:
        pass
    else:
        raise AssertionError("rc 2 must raise ValidationError")


def test_import_fails_loudly_without_library(tmp_path):
    """Copy the package without lib/ and import it: ImportError, no fallback."""
    import shutil

    pkg = tmp_path / "paper_2503_06823_b200"
    shutil.copytree(ROOT / "paper_2503_06823_b200", pkg, ignore=shutil.ignore_patterns("lib", "csrc"))
    code = "import paper_2503_06823_b200"
    r = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr, r.stderr[-500:]
