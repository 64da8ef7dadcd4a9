"""CPU: the C-ABI library loads and exports every symbol include/hire_cuda.h
declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hire_cuda.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^HIRE_API\s+[\w\s\*]+?\b(hire_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("hire_topk_run", "hire_topk_host", "hire_ffn_run", "hire_da_topk_run",
                 "hire_scorer_quantize", "hire_scorer_create_lowrank", "hire_comm_create"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2402_09360_b200 import _lib, build
    build.build()  # in-tree, no-op when fresh
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == declared()
    assert lib.hire_abi_version() == 1


def test_library_is_sm100a():
    from paper_2402_09360_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_error_path_without_gpu():
    """Argument validation runs before any device work: invalid calls fail
    with status 1 and the reference's message, even without a GPU."""
    from paper_2402_09360_b200 import _lib
    L = _lib.lib()
    h = ctypes.c_void_p()
    rc = L.hire_matrix_view(None, 4, 4, 0, ctypes.byref(h))
    assert rc == 1 and b"null" in L.hire_last_error()
