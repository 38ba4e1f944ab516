"""GPU: the reference's own C++ API, unchanged, next to the drop-in adapter
(include/groupot_b200.hpp) on the same ProblemInstance (oracle/dropin_check,
built from the reference headers in the build container)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "dropin_check")


@pytest.mark.skipif(not os.path.exists(EXE), reason="dropin_check not built (needs /root/reference)")
def test_reference_api_through_the_adapter():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    assert d["obj_rel"] <= 1e-9  # dual_objective
    assert d["grad_abs"] <= 1e-12  # dual_gradient (gradient entries ~1e-2)
    assert d["plan_eval_abs"] == 0.0  # recover_plan: bitwise
    # the reference's maximize() driving device evaluations through ObjectiveFn/GradientFn
    assert d["maximize_iters"][0] == d["maximize_iters"][1]
    assert d["maximize_x_abs"] <= 1e-8
    for mode in ("baseline", "fast", "fast-no-lb", "audit"):
        m = d[mode]
        assert m["converged"][0] == m["converged"][1]
        assert m["obj_rel"] <= 1e-6
        if m["converged"][0]:
            assert m["plan_abs"] <= 1e-6
    # the reference's maximize over the device's screened callbacks == solve_fast
    sm = d["screened_maximize"]
    assert sm["iters"][0] == sm["iters"][1] and sm["history_equal"] == 1
    assert sm["x_abs"] == 0.0 and sm["skipped"] > 0
    # audit_solve of fast_no_lower_bound options: no active set, exact order -> identical
    a = d["audit_nolb"]
    assert a["iters"][0] == a["iters"][1] and a["grad_calls"][0] == a["grad_calls"][1]
    assert a["in_active"] == [0, 0] and a["active_checks"] == [0, 0] and a["obj_equal"] == 1
    # run_grid (bench.hpp:137-180) on one warm device context, exact-order solves
    g = d["grid"]
    assert g["rows"] == [12, 12] and g["sink_calls"] == 12 and g["csv_roundtrip"] == 1
    assert g["ints_equal"] == 1 and g["obj_equal"] == 1 and g["sparsity_equal"] == 1
    assert g["res_abs"] <= 1e-12
    # CSV files -> load_csv -> the adapter's make_instance on the device
    c = d["csv_device"]
    assert c["iters"][0] == c["iters"][1] and c["x_equal"] == 1 and c["obj_equal"] == 1
    assert c["plan_abs"] == 0.0
    assert d["negative_cost_fields"] == 1 and d["marginal_fields"] == 1
    assert d["audit_violation"] == 1
