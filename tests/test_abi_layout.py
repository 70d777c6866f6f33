"""The ctypes binding's structures match include/ens.h field by field (CPU, no GPU).

A plain-C program compiled against the header prints sizeof and every field's offset of
ens_mesh, ens_materials, ens_options and ens_info; the ctypes Structures of _ffi.py must
agree, so that a field added to the header and not to the binding (or the reverse) fails
here instead of shifting every later field at run time.
"""
import os
import shutil
import subprocess

import pytest

from paper_2101_09059_b200 import _ffi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAIRS = [("ens_mesh", _ffi.EnsMesh), ("ens_materials", _ffi.EnsMaterials),
         ("ens_options", _ffi.EnsOptions), ("ens_info", _ffi.EnsInfo)]


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_ctypes_structures_match_header(tmp_path):
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "ens.h"', "int main(void) {"]
    for cname, cls in PAIRS:
        lines.append(f'    printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'    printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["    return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {(a, b): int(c) for a, b, c in (l.split() for l in out if l.strip())}
    for cname, cls in PAIRS:
        assert got[(cname, "sizeof")] == _ffi.C.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)
