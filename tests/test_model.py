"""Model-level caller: mlp_forward (model.cpp:115-127) on
the device against the reference's own mlp_forward (oracle/_ref)."""
import numpy as np
import pytest


def _layer_arrays(rng, m, n, r):
    w = rng.standard_normal((m, n)) * 0.1
    a = rng.standard_normal((m, r)) * 0.1
    b = rng.standard_normal((r, n)) * 0.1
    return w, a, b


@pytest.mark.gpu
@pytest.mark.parametrize("n,h,r,s", [(96, 160, 8, 0.5), (128, 352, 16, 0.3), (64, 64, 0, 1.0)])
def test_gpu_mlp_forward_matches_reference(reforacle, cuda, n, h, r, s):
    import torch
    import paper_2504_19449_b200 as rsp
    from paper_2504_19449_b200 import model
    rng = np.random.default_rng(n + h + r)
    mk = {}
    ref = {}
    for name, (m, k) in {"up": (h, n), "gate": (h, n), "down": (n, h)}.items():
        w, a, b = _layer_arrays(rng, m, k, r)
        mk[name] = rsp.DecomposedLayer(torch.from_numpy(w), torch.from_numpy(a) if r else None,
                                       torch.from_numpy(b) if r else None, rsp.SparsityPlan(s, r),
                                       weight_dtype="f32")
        W, A, B = mk[name].export()  # the stored (fp32-rounded) values feed the reference
        ref[name] = reforacle.layer(np.ascontiguousarray(W.T), A if r else np.zeros((m, 0)),
                                    B if r else np.zeros((0, k)), s)
    for t in range(3):
        x = rng.standard_normal(n).astype(np.float32)
        got = model.mlp_forward(torch.from_numpy(x).to(cuda), mk["up"], mk["gate"], mk["down"]).cpu().numpy()
        want = reforacle.mlp_forward(ref["up"], ref["gate"], ref["down"], x.astype(np.float64))
        assert np.max(np.abs(got - want)) <= 1e-4 * np.max(np.abs(want)), t


@pytest.mark.gpu
def test_gpu_mlp_forward_length_check(cuda):
    import torch
    import paper_2504_19449_b200 as rsp
    from paper_2504_19449_b200 import model
    up = rsp.DecomposedLayer(torch.randn(32, 16), None, None, rsp.SparsityPlan(1.0, 0), weight_dtype="f32")
    with pytest.raises(rsp.UsageError):
        model.mlp_forward(torch.randn(17, device=cuda), up, up, up)
