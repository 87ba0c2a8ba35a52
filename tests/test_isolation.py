"""The oracle and the CUDA path share no code (task rule ③): the product
package never imports, links or includes anything under oracle/, and the
oracle never includes product headers.  CPU only."""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1304_5553_b200")


def product_files():
    files = glob.glob(os.path.join(PKG, "**", "*.py"), recursive=True)
    files += glob.glob(os.path.join(PKG, "csrc", "*"))
    files += glob.glob(os.path.join(ROOT, "include", "*.h"))
    return files


def test_product_sources_do_not_reference_oracle():
    for f in product_files():
        src = open(f).read()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
        assert not re.search(r'#include\s+[<"].*oracle', src), f
        assert "liboracle" not in src, f


def test_oracle_does_not_include_product_code():
    for f in glob.glob(os.path.join(ROOT, "oracle", "*")):
        if f.endswith((".so", ".pyc")) or os.path.isdir(f):
            continue
        src = open(f).read()
        assert not re.search(r"^\s*(import|from)\s+paper_1304_5553_b200\b", src, re.M), f
        assert not re.search(r'#include\s+[<"].*(gpuarray\.h|ga_device|ga_host|scan_kernel)', src), f


def test_importing_product_does_not_load_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_1304_5553_b200, paper_1304_5553_b200.dist; "
            "print('oracle' in sys.modules)" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "False"


def test_product_library_does_not_link_oracle():
    lib = os.path.join(PKG, "libgpuarray.so")
    if not os.path.exists(lib):
        from conftest import product_build
        product_build()
    deps = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert "oracle" not in deps
    syms = subprocess.run(["nm", "-D", lib], capture_output=True, text=True).stdout
    assert "oracle_" not in syms


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without libgpuarray.so the package refuses to import."""
    import shutil
    shutil.copytree(PKG, tmp_path / "paper_1304_5553_b200",
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    code = "import sys; sys.path.insert(0, %r); import paper_1304_5553_b200" % str(tmp_path)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.returncode != 0
    assert "no CPU fallback" in out.stderr
