"""CPU checks of the BASELINE config generators (no GPU)."""

from paper_2504_19449_b200 import workloads as wl


def test_config4_plans_budget_and_clamps():
    # every feasible linear spends exactly (1 - sparsity) of dense by the reference io_cost
    for sp in (0.3, 0.4, 0.5, 0.6, 0.7):
        for r in (64, 128, 256, 512):
            plans, clamped = wl.config4_plans(sp, r, n_layers=1)
            assert len(plans) == 7
            for (name, m, n, s, rr) in plans:
                assert 0.0 <= s <= 1.0 and 0 <= rr <= min(m, n)
                cost = s + rr * (m + n) / (m * n)
                if s > 0.0:
                    assert abs(cost - (1.0 - sp)) < 1e-9
                else:
                    assert cost <= 1.0 - sp + 1e-12
            names = {c[0] for c in clamped}
            assert names <= {"k_proj", "v_proj"}
    # infeasible for k/v at r=256 / 70% and r=512 / 40..70%
    assert {c[0] for c in wl.config4_plans(0.7, 256, 1)[1]} == {"k_proj", "v_proj"}
    for sp in (0.4, 0.5, 0.6, 0.7):
        assert {c[0] for c in wl.config4_plans(sp, 512, 1)[1]} == {"k_proj", "v_proj"}
    assert wl.config4_plans(0.3, 512, 1)[1] == []
    assert wl.config4_plans(0.6, 256, 1)[1] == []
