"""The C-ABI library loads and exports every symbol include/ringmix_b200.h declares
(no CUDA call is made: this runs on the CPU-only build container)."""

from __future__ import annotations

import ctypes
import re
import subprocess

from conftest import ROOT

HEADER = ROOT / "include" / "ringmix_b200.h"


def declared_symbols() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(rm_[a-z0-9_]+)\s*\(", text))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for name in ("rm_perm_tables", "rm_perm_sequential", "rm_ring_mix_sgd_f32",
                 "rm_ring_mix_sgd_bf16", "rm_ring_mix_sgd_f64", "rm_mean_sgd_f32",
                 "rm_spsgd_f32", "rm_pcg_seed", "rm_pcg_permutations", "rm_last_error"):
        assert name in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2002_01119_b200 import _lib

    lib = _lib.load()
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    # and the binding table covers the same set
    assert set(_lib.exported_symbols()) | set(_lib.OPTIONAL_SIGNATURES) >= declared_symbols()


def test_library_is_sm100a_code():
    so = ROOT / "paper_2002_01119_b200" / "lib" / "libringmix_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_last_error_is_a_string_without_cuda():
    from paper_2002_01119_b200 import _lib

    assert isinstance(_lib.last_error(), str)
    # argument validation happens before any CUDA call
    lib = _lib.load()
    rc = lib.rm_perm_tables(None, 0, 0, 1, 0, None, None, None, None, None)
    assert rc == _lib.RM_EINVAL
    assert "n >= 1" in _lib.last_error()


def test_abi_uses_plain_c_types_only():
    code = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    assert "torch" not in code and "at::" not in code and "Tensor" not in code


def test_header_compiles_as_c_and_cpp(tmp_path):
    """A cgo / JNI / plain-C caller includes the header as C99; a C++ caller as C++."""
    import shutil
    import subprocess
    header = ROOT / "include" / "ringmix_b200.h"
    for cc, lang, std in (("gcc", "c", "-std=c99"), ("g++", "c++", "-std=c++17")):
        if shutil.which(cc) is None:
            continue
        r = subprocess.run([cc, "-fsyntax-only", "-Wall", "-Werror", "-x", lang, std, str(header)],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_plain_c_program_links_and_calls_the_library(tmp_path):
    """What a cgo / FFI binding does: a C program includes the header, links
    libringmix_b200.so and calls host-side entry points (no GPU needed for these)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        return
    src = tmp_path / "caller.c"
    src.write_text(
        "#include <stdio.h>\n"
        '#include "ringmix_b200.h"\n'
        "int main(void) {\n"
        "  int v = rm_version();\n"
        "  long long ws = (long long)rm_normal_workspace_bytes(4, 1000);\n"
        "  long long bad = (long long)rm_normal_workspace_bytes(0, 1000);\n"
        '  printf("%d %lld %lld\\n", v, ws, bad);\n'
        "  return (v > 0 && ws > 0 && bad < 0) ? 0 : 1;\n"
        "}\n")
    exe = tmp_path / "caller"
    lib = ROOT / "paper_2002_01119_b200" / "lib"
    r = subprocess.run(["gcc", "-std=c99", "-I", str(ROOT / "include"), str(src), "-L", str(lib),
                        "-lringmix_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.stdout, r.stderr)
