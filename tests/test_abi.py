"""The C-ABI library loads (no GPU needed) and exports every symbol that
include/ltfb_gpu.h declares; error codes map onto the reference taxonomy."""
import ctypes
import os
import re
import subprocess

import pytest

L = pytest.importorskip("paper_1910_02270_b200")
from paper_1910_02270_b200 import _lib  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(REPO, "include", "ltfb_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ltfb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_python_binds():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for s in declared_symbols():
        getattr(lib, s)


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_error_mapping_without_gpu():
    assert _lib.lib.ltfb_abi_version() == 1
    with pytest.raises(L.ContractError):
        L.partition_dataset([1, 2], 5, 0)
    with pytest.raises(L.ConfigError):
        L.SurrogateArch(hidden_act="swish").c()


def test_cpp_facade_compiles_and_links(tmp_path):
    """include/ltfb_b200/trainer.hpp (the C++ drop-in façade) compiles with
    the reference's C++20 toolchain and links against the library."""
    import os
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = os.path.join(repo, "tests", "cpp", "facade_test.cpp")
    lib_dir = os.path.dirname(L.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++20", "-O0", "-I" + os.path.join(repo, "include"), src, "-L" + lib_dir,
                        "-lltfb_gpu", "-o", str(tmp_path / "facade_test")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
