"""The C-ABI library loads and exports every symbol include/sph.h declares (CPU only:
no compute call is made without a GPU), and the ctypes structs match the header."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1404_2303_b200 as sphlib
from paper_1404_2303_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sph.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(sph_[a-z_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return sphlib.load()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 9
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(names) == set(sphlib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True).stdout
    for nm in names:
        assert re.search(rf"\bT {nm}\b", out), nm


def test_config_default_matches_paper_constants(lib):
    cfg = sphlib.default_config((2.0, 1.0, 1.0))
    assert cfg.abi_version == 2 and list(cfg.box) == [2.0, 1.0, 1.0]
    assert cfg.n_ngb == 48.0 and cfg.alpha == pytest.approx(0.8)
    assert cfg.gamma == pytest.approx(5 / 3)
    assert cfg.split_count == 300 and cfg.split_fraction == pytest.approx(0.875)
    assert cfg.flags & sphlib.SPH_F_SYNC


def test_struct_sizes_match_header(lib):
    # compile a tiny C program against the header and compare sizeof/offsetof
    code = r'''
#include <stdio.h>
#include <stddef.h>
#include "sph.h"
int main(){printf("%zu %zu %zu %zu %zu\n", sizeof(sph_config), sizeof(sph_stats),
 offsetof(sph_config, flags), offsetof(sph_config, slab_hi), offsetof(sph_stats, ms_build));return 0;}
'''
    tmp = os.path.join(ROOT, "build")
    os.makedirs(tmp, exist_ok=True)
    c = os.path.join(tmp, "abi_sizes.c")
    exe = os.path.join(tmp, "abi_sizes")
    open(c, "w").write(code)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
    got = list(map(int, subprocess.check_output([exe]).split()))
    assert got == [ctypes.sizeof(sphlib.Config), ctypes.sizeof(sphlib.Stats),
                   sphlib.Config.flags.offset, sphlib.Config.slab_hi.offset, sphlib.Stats.ms_build.offset]


def test_status_strings(lib):
    for s in range(-7, 1):
        assert lib.sph_status_string(s).decode().startswith("SPH_")


def test_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1404_2303_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", txt, flags=re.M), f
                assert "oracle/" not in txt.replace("`oracle/`", ""), f
