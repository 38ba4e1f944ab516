"""make_instance on the device (gsot_cost_matrix_device / gsot_create_features)
against the reference's make_instance from the same CSV files: cost matrix,
marginals and partition bitwise (normalised or not, uniform or weighted
marginals), and the device context built from the features evaluates and
solves exactly like one built from the reference's cost matrix."""
import os

import numpy as np
import pytest

import paper_2303_07597_b200 as G
from oracle_bindings import ref_available, ref_make_instance

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def write_pair(tmp_path, seed, m_per=(5, 3, 9, 1), n=23, d=4, weighted=False):
    rng = np.random.default_rng(seed)
    labels = np.repeat(np.arange(1, len(m_per) + 1), m_per)
    perm = rng.permutation(labels.size)  # unsorted on disk: load_csv sorts stably
    feats = rng.normal(size=(labels.size, d)) * 3.0
    sp, tp = os.path.join(tmp_path, "s.csv"), os.path.join(tmp_path, "t.csv")
    with open(sp, "w") as f:
        f.write("label" + (",weight" if weighted else "") + "".join(f",f{k}" for k in range(d)) + "\n")
        for i in perm:
            w = f",{rng.uniform(0.5, 2):.17g}" if weighted else ""
            f.write(f"{labels[i]}{w}," + ",".join(f"{v:.17g}" for v in feats[i]) + "\n")
    tf = rng.normal(size=(n, d)) * 3.0 + 0.5
    with open(tp, "w") as f:
        f.write(("weight," if weighted else "") + ",".join(f"f{k}" for k in range(d)) + "\n")
        for row in tf:
            w = f"{rng.uniform(0.5, 2):.17g}," if weighted else ""
            f.write(w + ",".join(f"{v:.17g}" for v in row) + "\n")
    return sp, tp


@pytest.mark.parametrize("normalize", [False, True])
@pytest.mark.parametrize("weighted", [False, True])
def test_make_instance_bitwise(tmp_path, normalize, weighted):
    sp, tp = write_pair(tmp_path, 3 + int(normalize) + 2 * int(weighted), weighted=weighted)
    src, tgt = G.load_csv(sp, tp)
    m, n = src.features.shape[0], tgt.features.shape[0]
    cost, a, b, sizes = ref_make_instance(sp, tp, m, n, normalize, weighted)
    inst = G.make_instance(src, tgt, normalize, weighted)
    assert np.array_equal(inst.cost, cost)
    assert np.array_equal(inst.a, a) and np.array_equal(inst.b, b)
    assert inst.groups.sizes() == sizes.tolist()
    # the context built from the features on the device (the cost never on
    # the host) evaluates bitwise like one built from the reference's cost
    p = G.RegParams(0.5, 0.4)
    c1 = G.make_device_instance(src, tgt, p, normalize, weighted)
    c2 = G.Context.from_arrays(cost, sizes, a, b, p.gamma(), p.mu())
    x = np.random.default_rng(1).uniform(0, 0.3, m + n)
    o1, g1, _ = c1.eval(x)
    o2, g2, _ = c2.eval(x)
    assert o1 == o2 and np.array_equal(g1, g2)
    r1 = c1.solve(mode=1, max_outer_loops=3, grad_tol=1e-12, exact=True)
    r2 = c2.solve(mode=1, max_outer_loops=3, grad_tol=1e-12, exact=True)
    assert np.array_equal(r1["x"], r2["x"]) and r1["objective"] == r2["objective"]
    c1.close()
    c2.close()


def test_device_instance_rejects_like_validate_instance(tmp_path):
    # a non-finite feature makes cost entries non-finite: NegativeCost with
    # the first offender in j-major order (core.hpp:118-123)
    sp, tp = write_pair(tmp_path, 9)
    src, tgt = G.load_csv(sp, tp)
    tgt.features[4, 1] = np.inf
    src.features[2, 0] = np.nan
    with pytest.raises(G.NegativeCost) as ei:
        G.make_device_instance(src, tgt, G.RegParams(1.0, 1.0))
    assert (ei.value.row, ei.value.col) == (2, 0)  # j-major: column 0, row 2 comes first
