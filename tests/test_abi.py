"""The C-ABI library loads and exports every symbol include/cc.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_1607_06156_b200 import build as ccbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(cc_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    ccbuild.build()
    import paper_1607_06156_b200 as cc
    return cc.lib()


def test_header_parses():
    names = declared_functions()
    for must in ("cc_init", "cc_load_edges", "cc_run", "cc_labels_u32", "cc_labels_u64", "cc_destroy"):
        assert must in names


def test_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_names_cover_header():
    import paper_1607_06156_b200 as cc
    assert set(declared_functions()) <= set(cc.EXPORTS)


def test_host_only_entry_points(lib):
    assert lib.cc_version().startswith(b"cc-b200")
    assert lib.cc_status_string(2) == b"CC_ERR_RANGE"
    # NULL arguments are rejected with a status, never a crash
    assert lib.cc_init(None, None) == 1
    assert lib.cc_run(None, 0, None) == 1
    assert lib.cc_destroy(None) == 1


def test_struct_layout_matches_header():
    """ctypes mirrors of cc_config / cc_report have the C sizes (compiled probe)."""
    import subprocess
    import tempfile
    import paper_1607_06156_b200 as cc
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "cc.h"
int main(){printf("%zu %zu %zu %zu\n", sizeof(cc_config), sizeof(cc_report), sizeof(cc_iter_stat),
 offsetof(cc_report, iters));return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        sizes = list(map(int, subprocess.check_output([exe]).split()))
    assert sizes == [ctypes.sizeof(cc.cc_config), ctypes.sizeof(cc.cc_report),
                     ctypes.sizeof(cc.cc_iter_stat), cc.cc_report.iters.offset]


def test_bench_reference_arm_prints_contract_line():
    """bench.py --impl reference (the oracle arm) runs on CPU and prints one JSON line with
    the contract's keys (small config to keep the CPU suite fast)."""
    import json
    import subprocess
    import sys
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                                   "--config", "c1", "--steps", "2", "--warmup", "1"], text=True,
                                  cwd=ROOT, timeout=600)
    line = json.loads(out.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_unique_id_host_only(lib):
    """cc_get_unique_id: 128 bytes from the NCCL the library loads at run time
    (no GPU needed); NULL output is rejected with a status."""
    import paper_1607_06156_b200 as cc
    assert lib.cc_get_unique_id(None, None, 0) == 1
    try:
        a = cc.cc_get_unique_id()
    except cc.CCError as e:  # no usable NCCL / network interface in this container
        pytest.skip(str(e))
    assert isinstance(a, bytes) and len(a) == cc.CC_UNIQUE_ID_BYTES
    assert a != cc.cc_get_unique_id()
