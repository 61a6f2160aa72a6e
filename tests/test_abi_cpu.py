"""The C-ABI library builds for sm_100a, loads without a GPU and exports every symbol that
include/ffs.h declares (no compute calls: there is no GPU here)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ffs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ffs_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("ffs_sample", "ffs_sample_marginal", "ffs_workspace_bytes", "ffs_debug_trace",
              "ffs_last_error", "ffs_sample_host"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    torch = pytest.importorskip("torch")  # noqa: F841  (binding imports torch)
    from paper_2109_07358_b200 import ffs
    lib = ffs.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(ffs.EXPORTED)


def test_sass_is_sm100a_and_uses_fp64_pipe():
    import shutil
    import subprocess
    from paper_2109_07358_b200 import build
    so = build.build()
    if shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("no cuobjdump")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-lelf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([exe, "-sass", so], capture_output=True, text=True).stdout
    assert "DFMA" in sass


def test_no_cpu_fallback_in_product_path():
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_2109_07358_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "ffs_ref" not in txt, f


def test_option_table_matches_header():
    """The binding's option names map to the values of include/ffs.h's ffs_option enum."""
    pytest.importorskip("torch")
    from paper_2109_07358_b200 import ffs
    src = open(os.path.join(ROOT, "include", "ffs.h")).read()
    enum = dict((n.lower(), int(v)) for n, v in re.findall(r"FFS_OPT_([A-Z0-9_]+)\s*=\s*(\d+)", src))
    last = enum.pop("last")
    assert last == max(enum.values())
    assert sorted(enum.values()) == list(range(1, last + 1))
    assert {k: v for k, v in ffs.OPTIONS.items()} == enum


def test_sass_has_the_blackwell_tensor_path():
    """The Ozaki GEMM is tcgen05 code: UTCIMMA (tcgen05.mma.kind::i8), UTMALDG (TMA loads), LDTM
    (tcgen05.ld) appear in the library's SASS."""
    import shutil
    import subprocess
    from paper_2109_07358_b200 import build
    so = build.build()
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("no cuobjdump")
    sass = subprocess.run([exe, "-sass", so], capture_output=True, text=True).stdout
    for mnem in ("UTCIMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem
