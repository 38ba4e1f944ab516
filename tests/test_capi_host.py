"""CPU: the C-ABI library loads and exports what include/gsot.h declares; the
host-side mirror of the reference API enforces the reference's argument
checks; without a GPU every compute entry point fails loudly (no CPU
fallback); the product's instance generator equals the oracle's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2303_07597_b200 as G
from paper_2303_07597_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "gsot.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"GSOT_API\s+[\w\s\*]+?\b(gsot_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 29
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding declares a signature for each of them
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    so = _lib.LIB_PATH
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                       text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout


def test_version_string():
    assert b"sm_100a" in _lib.lib().gsot_version()


def cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    inst = G.ProblemInstance(np.zeros((2, 2)), [0.5, 0.5], [0.5, 0.5], G.GroupPartition([2]))
    with pytest.raises(G.CudaError):
        G.dual_objective(G.DualState(np.zeros(2), np.zeros(2)), inst, G.RegParams(1, 1))
    h = C.c_void_p()
    cost = np.zeros((2, 2), order="F")
    st = _lib.lib().gsot_create(cost.ctypes.data_as(C.c_void_p), 2, 2,
                                np.array([2], np.int32).ctypes.data_as(C.c_void_p), 1,
                                np.array([.5, .5]).ctypes.data_as(C.c_void_p),
                                np.array([.5, .5]).ctypes.data_as(C.c_void_p), 1.0, 1.0,
                                C.byref(h))
    assert st == 8 and not h.value  # GSOT_ERR_CUDA, no context


def test_params_from_rho():
    # test_core.cpp:83-102
    p1 = G.params_from_rho(1.0, 0.5)
    assert (p1.gamma(), p1.mu(), p1.tau()) == (0.5, 1.0, 0.5)
    p2 = G.params_from_rho(10.0, 0.8)
    assert abs(p2.gamma() - 2.0) <= 1e-15 and abs(p2.mu() - 4.0) <= 1e-14
    assert abs(p2.tau() - 8.0) <= 1e-14
    for rho in (0.0, 1.0, -0.2, 1.3):
        with pytest.raises(G.RhoOutOfRange) as ei:
            G.params_from_rho(1.0, rho)
        # errors.hpp:49-56: the field and the message of RhoOutOfRange(rho)
        assert ei.value.rho == rho
        assert str(ei.value) == f"rho = {rho:.6f} is outside the open interval (0,1)"
    with pytest.raises(G.Error):
        G.RegParams(0.0, 1.0)
    with pytest.raises(G.Error):
        G.RegParams(1.0, -1.0)


def test_group_partition():
    # test_core.cpp:8-21
    gp = G.GroupPartition([2, 3, 1])
    assert gp.num_groups() == 3 and gp.total_size() == 6
    assert [gp.offset(l) for l in range(3)] == [0, 2, 5] and gp.size(1) == 3
    assert gp.offsets() == [0, 2, 5, 6]
    for bad in ([], [2, 0], [-1]):
        with pytest.raises(G.PartitionMismatch):
            G.GroupPartition(bad)


def test_dimension_checks_precede_device_work():
    inst = G.ProblemInstance(np.zeros((3, 2)), np.full(3, 1 / 3), [0.5, 0.5],
                             G.GroupPartition([3]))
    bad = G.DualState(np.zeros(2), np.zeros(2))
    with pytest.raises(G.DimensionMismatch):
        G.dual_objective(bad, inst, G.RegParams(1.0, 1.0))
    with pytest.raises(G.DimensionMismatch):
        G.dual_gradient(bad, inst, G.RegParams(1.0, 1.0))
    with pytest.raises(G.DimensionMismatch):
        G.recover_plan(bad, inst, G.RegParams(1.0, 1.0))
    with pytest.raises(G.DimensionMismatch) as ei:
        G.validate_instance(G.ProblemInstance(np.zeros((3, 2)), [1.0], [0.5, 0.5],
                                              G.GroupPartition([3])))
    assert str(ei.value) == "dimension mismatch: marginal a has length 1, cost has 3 rows"
    # core.hpp:117-131: the cost scan precedes the length checks, so a
    # negative entry wins over a wrong-length marginal (first offender j-major)
    cost = np.zeros((3, 2))
    cost[2, 0], cost[0, 1] = -1.0, -2.0
    with pytest.raises(G.NegativeCost) as ei:
        G.validate_instance(G.ProblemInstance(cost, [1.0], [0.5, 0.5], G.GroupPartition([3])))
    assert (ei.value.row, ei.value.col, ei.value.value) == (2, 0, -1.0)
    assert str(ei.value) == "cost(2,0) = -1.000000 is negative or non-finite"


def test_cost_is_frozen():
    inst = G.ProblemInstance(np.zeros((2, 2)), [0.5, 0.5], [0.5, 0.5], G.GroupPartition([2]))
    with pytest.raises(ValueError):
        inst.cost[0, 0] = 1.0


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_generator_matches_oracle(oracle, cfg):
    m, n, L, d = G.config_shape(cfg)
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    s2, t2 = np.empty((m, d)), np.empty((n, d))
    z2, a2, b2 = np.empty(L, np.int32), np.empty(m), np.empty(n)
    oracle.lib.go_config_features(C.c_int(cfg), C.c_uint64(cfg),
                                  *[v.ctypes.data_as(C.c_void_p) for v in (s2, t2, z2, a2, b2)])
    assert np.array_equal(src, s2) and np.array_equal(tgt, t2)
    assert np.array_equal(sizes, z2) and np.array_equal(a, a2) and np.array_equal(b, b2)
    assert sizes.sum() == m and sizes.min() >= 2
    assert abs(oracle.lib.go_compensated_sum(a, m) - 1.0) <= 1e-12


def test_config4_zipf_sizes():
    src, tgt, sizes, a, b = G.config_features(4, 4)
    assert sizes.max() == 4000 and sizes.min() == 9 and int(np.median(sizes)) == 20
    assert np.all(np.diff(sizes) <= 0) or sizes[1] >= sizes[2]
    assert (a > 0).all() and abs(a.sum() - 1.0) < 1e-12  # Dirichlet(1) weights
