"""CPU checks of the C-ABI boundary: libqvts.so loads and exports every symbol include/qvts.h
declares; descriptor validation happens before any CUDA call.  No compute calls."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qvts.h")


@pytest.fixture(scope="module")
def qlib():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1810_00204_b200", "csrc")], check=True,
                   stdout=subprocess.DEVNULL)
    from paper_1810_00204_b200 import qvts
    return qvts


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"QVTS_API\s+[\w\s\*]*?\b(qvts_\w+)\s*\(", text)))


def test_header_declares_the_five_north_star_calls():
    syms = declared_symbols()
    for s in ("qvts_model_create", "qvts_value_iteration", "qvts_belief_update", "qvts_plan_step",
              "qvts_run_episodes"):
        assert s in syms


def test_library_exports_every_declared_symbol(qlib):
    L = C.CDLL(qlib.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", qlib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(qvts_\w+)\b", out))
    assert set(declared_symbols()) == exported


def test_binding_names_match_abi(qlib):
    for s in declared_symbols():
        assert hasattr(qlib, s) or s == "qvts_model_destroy", s


def test_library_is_sm100a(qlib):
    out = subprocess.run(["cuobjdump", "--list-elf", qlib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("bad", [
    dict(goal=0),                       # goal on an occupied cell
    dict(p_intended=0.9),               # noise does not sum to 1
    dict(sensor_acc=0.5),
    dict(gamma=1.0),
])
def test_invalid_descriptor_rejected_before_cuda(qlib, bad):
    occ = np.zeros(9, np.uint8)
    occ[0] = 1
    kw = dict(goal=4, action_mask=0x1FF, p_intended=0.8, p_stay=0.1, p_lateral=0.05, sensor_acc=0.95, gamma=0.95)
    kw.update(bad)
    with pytest.raises(qlib.QvtsError) as e:
        qlib.qvts_model_create(3, 3, occ, **kw)
    assert e.value.code == 2    # QVTS_ERR_INVALID_MODEL


def test_unsupported_action_mask(qlib):
    with pytest.raises(qlib.QvtsError) as e:
        qlib.qvts_model_create(3, 3, np.zeros(9, np.uint8), 4, action_mask=0x003)
    assert e.value.code == 1
