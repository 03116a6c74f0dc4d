"""CPU suite: libtidq.so loads and exports every entry point include/*.h
declares; the ctypes binding covers exactly that set.  No compute calls."""

import ctypes
import glob
import os
import re

import pytest

from paper_1807_01409_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(tidq_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_entry_points():
    names = declared_symbols()
    assert {"tidq_ctx_create", "tidq_store_upload", "tidq_scan", "tidq_last_error"} <= names


def test_library_builds_and_exports_all_declared_symbols():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_1807_01409_b200.build import build
        build()
    cdll = _lib.load()
    missing = [n for n in sorted(declared_symbols()) if not hasattr(cdll, n)]
    assert not missing, f"not exported: {missing}"


def test_binding_matches_header():
    assert set(_lib.exported_symbols()) == declared_symbols()


def test_abi_version_and_error_string():
    cdll = _lib.load()
    assert cdll.tidq_abi_version() == 1
    # a failing call sets a message without a GPU (null output pointer)
    rc = cdll.tidq_ctx_create(0, None)
    assert rc == _lib.E_INVALID
    assert b"null" in cdll.tidq_last_error()


def test_struct_layout_matches_header(tmp_path):
    """sizeof/offsetof of the ABI structs as gcc lays them out == ctypes."""
    import shutil
    import subprocess

    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    checks = {
        "tidq_synth_params": (_lib.SynthParams, ["n_triples", "base_index", "seed", "n_p", "n_e"]),
        "tidq_stream_spec": (_lib.StreamSpec, [f for f, _ in _lib.StreamSpec._fields_]),
        "tidq_scan_spec": (_lib.ScanSpec, ["n_keys", "keys", "n_streams", "streams", "flags", "write_counts"]),
        "tidq_convert_report": (_lib.ConvertReport, [f for f, _ in _lib.ConvertReport._fields_]),
    }
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "tidq.h"', "int main(void){"]
    for st, (_, fields) in checks.items():
        src.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fields:
            src.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    src.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True,
                                                               text=True, check=True).stdout.split("\n") if line)
    for st, (cls, fields) in checks.items():
        assert int(out[st]) == ctypes.sizeof(cls), st
        for f in fields:
            assert int(out[f"{st}.{f}"]) == getattr(cls, f).offset, f"{st}.{f}"


def test_product_never_imports_the_oracle():
    """oracle/ is test infrastructure: the package (and tools/) must not
    import it; there is no CPU fallback on the product path."""
    offenders = []
    for d in ("paper_1807_01409_b200", "tools"):
        for f in glob.glob(os.path.join(ROOT, d, "**", "*.py"), recursive=True):
            text = open(f).read()
            if re.search(r"^\s*(from\s+oracle\b|import\s+oracle\b)", text, flags=re.M):
                offenders.append(os.path.relpath(f, ROOT))
    assert not offenders, offenders


def test_python_constants_match_header_defines():
    """Every TIDQ_* integer #define the binding mirrors (flags, output kinds,
    error codes, limits) has the header's value."""
    text = open(os.path.join(ROOT, "include", "tidq.h")).read()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"^#define TIDQ_(\w+)\s+\(?(-?\d+)u?\)?", text, re.M)}
    mirrored = {k: v for k, v in defs.items() if hasattr(_lib, k)}
    assert {"SCAN_ASYNC", "SCAN_CONCAT", "OUT_LOCAL"} <= set(mirrored), sorted(mirrored)
    for k, v in mirrored.items():
        assert getattr(_lib, k) == v, k
