"""The ctypes mirrors of the C-ABI structs (paper_2110_13526_b200/_lib.py) agree with
include/cbct.h field by field: a tiny C program compiled against the header prints sizeof and
every offsetof, which must equal the ctypes layout.  Needs gcc only (no GPU, no libcbct)."""

import pathlib
import shutil
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_ctypes_structs_match_header(tmp_path):
    from paper_2110_13526_b200._lib import Geometry, PlanInfo

    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cbct.h"', "int main(void) {"]
    for cname, py in (("cbct_geometry", Geometry), ("cbct_plan_info", PlanInfo)):
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for field, _ in py._fields_:
            lines.append(f'printf("{cname} {field} %zu\\n", offsetof({cname}, {field}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        cname, field, value = line.split()
        got[(cname, field)] = int(value)
    for cname, py in (("cbct_geometry", Geometry), ("cbct_plan_info", PlanInfo)):
        assert got[(cname, "sizeof")] == ctypes_sizeof(py), cname
        for field, _ in py._fields_:
            assert got[(cname, field)] == getattr(py, field).offset, (cname, field)


def ctypes_sizeof(t):
    import ctypes

    return ctypes.sizeof(t)
