"""CPU-side checks of the boundary: libpf.so loads and exports every symbol include/pf.h declares,
the binding exposes the same names, and the product package never touches the oracle."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1501_07844_b200 as pf
    lib = ctypes.CDLL(pf.LIB_PATH)
    decl = _declared()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
        assert hasattr(pf, name), f"binding lacks {name}"
    assert sorted(pf.EXPORTED) == decl


def test_version_without_gpu():
    import paper_1501_07844_b200 as pf
    assert "sm_100a" in pf.pf_version()


def test_product_does_not_reference_oracle():
    pkg = os.path.join(ROOT, "paper_1501_07844_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b", text), f"{f} mentions the oracle"


def test_kernel_binary_is_sm100a():
    import subprocess
    import paper_1501_07844_b200 as pf
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pf.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_library_carries_nvtx_ranges():
    """The library marks its phases for nsys (boundary / interior / check / IPC step): NVTX range names."""
    import paper_1501_07844_b200 as pf
    data = open(pf.LIB_PATH, "rb").read()
    for name in (b"pf boundary", b"pf interior", b"pf check (residual read)", b"pf ipc step", b"pf_iterate"):
        assert name in data, name
