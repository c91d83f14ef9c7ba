"""Host-side checks of the C ABI (-m "not gpu"): the library builds and loads without a GPU,
exports every symbol include/prs.h declares, and its host-only logic behaves."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

import paper_2502_08370_b200 as prs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "prs.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(prs_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    prs.build()
    L = ctypes.CDLL(prs.SO)
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(L, name), name
    assert sorted(prs.EXPORTS) == syms


def test_struct_layout_matches_header():
    # field order and types of prs_problem as declared in include/prs.h
    text = open(os.path.join(ROOT, "include", "prs.h")).read()
    body = text[text.index("typedef struct prs_problem"):text.index("} prs_problem;")]
    fields = re.findall(r"^\s*(int|double)\s+([a-zA-Z_]+);", body, flags=re.M)
    names = [f for _, f in fields]
    assert names == [f for f, _ in prs.prs_problem._fields_]
    for (ty, name), (fname, cty) in zip(fields, prs.prs_problem._fields_):
        assert (cty is ctypes.c_double) == (ty == "double"), name


@pytest.mark.parametrize("N,P", [(8, 1), (8, 2), (8, 8), (64, 8), (32, 3), (7, 4), (5, 5)])
def test_partition_covers_slices_in_rank_order(N, P):
    nxt = 0
    for r in range(P):
        first, count = prs.partition(N, P, r)
        assert first == nxt and count >= 1
        nxt += count
    assert nxt == N
    counts = [prs.partition(N, P, r)[1] for r in range(P)]
    assert max(counts) - min(counts) <= 1


def test_partition_rejects_bad_arguments():
    for args in [(0, 1, 0), (4, 0, 0), (4, 2, 2), (4, 8, 0), (4, 2, -1)]:
        with pytest.raises(prs.PrsError):
            prs.partition(*args)


def test_create_rejects_invalid_configs_before_touching_the_gpu():
    import synth
    bad = [synth.Problem(dim=4), synth.Problem(n=0), synth.Problem(N=0), synth.Problem(G=7),
           synth.Problem(split=1, n=30, dd_strips=8), synth.Problem(split=1, n=32, dd_strips=4,
                                                                    dd_overlap=3)]
    for p in bad:
        with pytest.raises(prs.PrsError) as ei:
            prs.Context(p)
        assert ei.value.code == prs.PRS_EINVAL
    for p in [synth.Problem(dim=3, G=synth.DR), synth.Problem(dim=3, coef=1),
              synth.Problem(coef=2, split=0, n=32)]:  # mixed derivatives: DD split only
        with pytest.raises(prs.PrsError) as ei:
            prs.Context(p)
        assert ei.value.code == prs.PRS_EUNSUPPORTED


C_SMOKE = os.path.join(ROOT, "tests", "c", "abi_smoke.c")


def build_c_smoke(out_dir):
    """gcc a plain C client against include/prs.h and libprs.so (rpath to the in-tree library)."""
    import subprocess
    prs.build()
    exe = os.path.join(out_dir, "abi_smoke")
    libdir = os.path.dirname(prs.SO)
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           C_SMOKE, "-o", exe, os.path.join(prs.SO), f"-Wl,-rpath,{libdir}", "-lm"])
    return exe


def test_c_client_compiles_and_links_against_the_header(tmp_path):
    """A C program (tests/c/abi_smoke.c) compiles with -Wall -Werror against include/prs.h and
    links against libprs.so: the ABI is usable without Python."""
    exe = build_c_smoke(str(tmp_path))
    assert os.access(exe, os.X_OK)
