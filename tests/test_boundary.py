"""The drop-in boundary: the C-ABI library loads and exports every symbol the
header declares; the product never imports the oracle; no CPU fallback."""
import ast
import ctypes
import os

from paper_2502_09922_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2502_09922_b200")


def test_library_exports_every_header_symbol():
    syms = N.header_symbols()
    assert len(syms) >= 30
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares every header function too
    assert sorted(N.SIGNATURES) == syms


def test_library_reports_version_without_gpu():
    assert N.lib().lp_version() >= 100
    assert isinstance(N.lib().lp_last_error(), bytes)


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                elif isinstance(node, ast.ImportFrom):
                    assert (node.module or "").split(".")[0] != "oracle", f


def test_no_forbidden_batch_memcpy_calls():
    bad = ["cudaMemcpy" + "BatchAsync", "cudaMemcpy3D" + "BatchAsync", "cuMemcpy" + "BatchAsync",
           "cuMemcpy3D" + "BatchAsync"]
    for dirpath, _, files in os.walk(ROOT):
        if ".git" in dirpath or "gpurun_out" in dirpath:
            continue
        for f in files:
            if f.endswith((".cu", ".cuh", ".cpp", ".c", ".h", ".py")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                for b in bad:
                    assert b not in text, (f, b)
