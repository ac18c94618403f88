"""CPU checks of the boundary: libhelios.so builds for sm_100a, loads, exports every symbol that
include/helios.h declares, and its host-only logic (bounds, argument validation) behaves."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def so():
    from paper_2310_00837_b200 import build as hb
    return hb.build()


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "helios.h")).read()
    return sorted(set(re.findall(r"\b(helios_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(so):
    out = subprocess.check_output(["nm", "-D", "--defined-only", so], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if l.strip()}
    decl = declared_symbols()
    assert len(decl) >= 18
    missing = [s for s in decl if s not in exported]
    assert not missing, missing


def test_sm100a_cubin(so):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], text=True)
    assert "sm_100a" in out


def test_binding_names_match_header(so):
    from paper_2310_00837_b200 import helios as H
    assert sorted(H.ABI_SYMBOLS) == declared_symbols()
    assert H.helios_abi_version() == 2


def test_host_side_bounds_and_validation(so):
    from paper_2310_00837_b200 import helios as H
    mx, lvl, edg = H.helios_sample_bounds(1024, [15, 10, 5], 111_000_000, 1_600_000_000)
    assert lvl == [1024, 16384, 180224, 1081344] and edg == [15360, 163840, 901120] and mx == 1081344
    mx, lvl, edg = H.helios_sample_bounds(256, [10, 5], 10_000, 200_000)
    assert lvl == [256, 2816, 10_000] and mx == 10_000
    with pytest.raises(H.HeliosError) as e:
        H.helios_sample_bounds(4, [0], 10, 10)
    assert e.value.name == "E_INVALID"
    # CSR checks that happen before any device call
    with pytest.raises(H.HeliosError) as e:
        H.helios_graph_load(np.array([1, 2, 3]), np.array([0, 1, 1], dtype=np.int32))
    assert e.value.name == "E_INVALID"
