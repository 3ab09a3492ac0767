"""The C-ABI library loads on a CPU host and exports every symbol include/*.h declares.

No compute calls here (no GPU in the CPU suite); host-only entry points
(splatt_partition, splatt_version) are exercised, and device calls must fail
cleanly with a status, not crash.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from tests.conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "splatt_b200.h")


@pytest.fixture(scope="module")
def L():
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as sb
    return sb.lib()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(splatt_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    fns = declared_functions()
    for name in ("splatt_csf_build", "splatt_mttkrp", "splatt_cpd_als"):
        assert name in fns


def test_every_declared_symbol_is_exported(L):
    fns = declared_functions()
    assert len(fns) >= 14
    for name in fns:
        assert hasattr(L, name), name


def test_library_is_sm100a_and_no_oracle_link(L):
    import paper_1812_05961_b200 as sb
    assert "sm_100a" in sb.version()
    blob = open(sb.LIB_PATH, "rb").read()
    assert b"oracle_" not in blob  # the product never links the oracle


def test_partition_host_examples_and_agrees_with_oracle(L):
    import paper_1812_05961_b200 as sb
    for case in golden("spec_partition.json")["cases"]:
        assert sb.partition(case["weights"], case["G"]).tolist() == case["bounds"]
    rng = np.random.default_rng(0)
    for _ in range(200):
        w = rng.integers(0, 1000, int(rng.integers(1, 300))) ** 2
        G = int(rng.integers(1, 9))
        assert sb.partition(w, G).tolist() == oracle.partition(w, G).tolist()


def test_bad_args_return_status_without_device(L):
    p = C.c_void_p()
    st = L.splatt_ctx_create(C.byref(p), 0, None)
    if st == 0:  # a GPU is present: nothing to check here
        L.splatt_ctx_destroy(p)
        return
    assert st in (-1, -4)
    assert L.splatt_ctx_create(None, 0, None) == -1
    assert L.splatt_mttkrp(None, None, 0, None, 1, 1, None) == -1
    assert L.splatt_cpd_als(None, None, 1, 1, 0.0, 0, None) == -1
    assert L.splatt_partition(None, 0, 0, None) == -1
    assert L.splatt_mttkrp_csf(None, None, 0, 0, None, 1, 1, None) == -1
    assert L.splatt_csf_dispatch(None, 0, None, None, None) == -1
    assert L.splatt_ctx_set_exchange(None, 0) == -1
    assert L.splatt_ctx_set_partition(None, 0) == -1


def test_exchange_constants_match_header_and_binding():
    txt = open(HEADER).read()
    assert re.search(r"SPLATT_XCHG_COLLECTIVE\s*=\s*0\b", txt)
    assert re.search(r"SPLATT_XCHG_PEER\s*=\s*1\b", txt)
    src = open(os.path.join(ROOT, "paper_1812_05961_b200", "__init__.py")).read()
    assert '{"collective": 0, "peer": 1}' in src
    # the statistics struct ends with the exchange word in both the header and the binding
    assert re.search(r"int32_t\s+exchange;[^}]*}\s*splatt_stats;", txt, re.S)
    import paper_1812_05961_b200 as sb
    assert sb.Stats._fields_[-1][0] == "exchange"


def test_policy_constants_match_header():
    import paper_1812_05961_b200 as sb
    txt = open(HEADER).read()
    for name, val in (("ALL", sb.CSF_ALL), ("ONE", sb.CSF_ONE), ("TWO", sb.CSF_TWO)):
        assert re.search(rf"SPLATT_CSF_{name}\s*=\s*{val}\b", txt), name


def test_no_cpu_fallback_in_binding():
    src = open(os.path.join(ROOT, "paper_1812_05961_b200", "__init__.py")).read()
    assert "import oracle" not in src and "from oracle" not in src
