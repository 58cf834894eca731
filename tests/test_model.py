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


# ----------------------------------------------------------------------------- toy decoder (model.cpp:159-269)
def _toy(reforacle, tmp_path, layers=2):
    path = str(tmp_path / "toy.rspw")
    reforacle.model_write(path, num_layers=layers, embed=64, hidden=172, heads=4, vocab=256, seed=1, max_seq=64)
    return path


def _decomposed(model, reforacle, seed=0, weight_dtype="f32"):
    """One DecomposedLayer per linear (truncated-SVD factors, varied plans)
    plus the reference layers built from the exact values the device holds."""
    import torch
    import paper_2504_19449_b200 as rsp
    rng = np.random.default_rng(seed)
    ours, refs = [], []
    for idx in range(model.num_linear_layers()):
        w = model.linear_weight(idx)
        m, n = w.shape
        s, r = float(rng.uniform(0.2, 0.6)), int(rng.integers(4, 17))
        U, S, Vh = torch.linalg.svd(w, full_matrices=False)
        a, b = U[:, :r] * S[:r].sqrt(), S[:r].sqrt()[:, None] * Vh[:r]
        layer = rsp.DecomposedLayer(w, a, b, rsp.SparsityPlan(s, r), weight_dtype=weight_dtype)
        W, A, B = layer.export()
        ours.append(layer)
        refs.append(reforacle.layer(np.ascontiguousarray(W.T), A, B, s))
    return ours, refs


def test_read_rspw_host_parse(reforacle, tmp_path):
    from paper_2504_19449_b200 import model as M
    import paper_2504_19449_b200 as rsp
    path = _toy(reforacle, tmp_path)
    tm = M.ToyModel.read_rspw(path, device="cpu")
    assert tm.config.num_layers == 2 and tm.config.embed_dim == 64 and tm.config.hidden_dim == 172
    assert tuple(tm.blocks[1]["down"].shape) == (64, 172) and tm.num_linear_layers() == 14
    raw = open(path, "rb").read()
    bad = tmp_path / "bad.rspw"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(rsp.IoError):
        M.ToyModel.read_rspw(str(bad), device="cpu")
    bad.write_bytes(raw[:1000])
    with pytest.raises(rsp.IoError):
        M.ToyModel.read_rspw(str(bad), device="cpu")


@pytest.mark.gpu
def test_gpu_model_forward_and_perplexity_match_reference(reforacle, cuda, tmp_path):
    """model_forward / perplexity (model.cpp:159-269) with every decode-region
    linear on the R-Sparse kernels (q/k/v and the gated MLP as stack launches,
    down's input formed in-kernel) against the reference on the same model
    file and the same stored factor values."""
    from paper_2504_19449_b200 import model as M
    path = _toy(reforacle, tmp_path)
    tm = M.ToyModel.read_rspw(path, device=cuda)
    ours, refs = _decomposed(tm, reforacle)
    rng = np.random.default_rng(3)
    tok = rng.integers(0, 256, 24).tolist()
    for split in (0, 12):
        got = M.model_forward(tm, tok, ours, decode_start=split).cpu().numpy()
        want = reforacle.model_logits(path, tok, refs, decode_start=split)
        assert np.max(np.abs(got - want)) <= 1e-4 * np.max(np.abs(want)), split
    dense = M.model_forward(tm, tok).cpu().numpy()
    assert np.max(np.abs(dense - reforacle.model_logits(path, tok))) <= 1e-9 * np.max(np.abs(dense))
    ppl = M.perplexity(tm, tok, 12, ours)
    want = reforacle.model_perplexity(path, tok, 12, refs)
    assert abs(ppl - want) <= 1e-5 * want, (ppl, want)


@pytest.mark.gpu
def test_gpu_recipe_evaluator_loss_matches_reference(reforacle, cuda, tmp_path):
    """RecipeEvaluator::loss (search.cpp:90-97): scores from the dense model's
    calibration inputs, decompose_with_svd at Recipe::plan_for, mean
    perplexity -- cuSOLVER SVD here, the reference's Jacobi SVD there."""
    import paper_2504_19449_b200 as rsp
    from paper_2504_19449_b200 import model as M
    path = _toy(reforacle, tmp_path)
    tm = M.ToyModel.read_rspw(path, device=cuda)
    rng = np.random.default_rng(5)
    calib = rng.integers(0, 256, 64).tolist()
    rho = rng.uniform(0.3, 0.7, 14).tolist()
    budget = [0.5] * 14
    ev = M.RecipeEvaluator(tm, calib, 32)
    got = ev.loss(rsp.Recipe(rho, budget))
    want, want_dense = reforacle.recipe_loss(path, calib, 32, rho, budget)
    assert abs(got - want) <= 1e-4 * want, (got, want)
    assert abs(ev.dense_loss() - want_dense) <= 1e-9 * want_dense


@pytest.mark.gpu
def test_gpu_gated_mlp_stack_matches_unfused(cuda):
    """RSP_XOP_SILU_GATE: the MLP as one stack launch (gate | up, then down
    with up * silu(gate) formed in its x load) equals the unfused chain."""
    import torch
    import paper_2504_19449_b200 as rsp
    from paper_2504_19449_b200 import model as M
    rng = np.random.default_rng(9)
    n, h = 512, 1376
    mk = lambda m, k, s, r: rsp.DecomposedLayer(torch.randn(m, k, device=cuda) * 0.05,  # noqa: E731
                                                torch.randn(m, r, device=cuda) * 0.1,
                                                torch.randn(r, k, device=cuda) * 0.1, rsp.SparsityPlan(s, r),
                                                weight_dtype="f32")
    up, gate, down = mk(h, n, 0.3, 40), mk(h, n, 0.25, 48), mk(n, h, 0.2, 64)
    u = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(cuda)
    yug = torch.zeros(2 * h, device=cuda)
    yd = torch.zeros(n, device=cuda)
    st = rsp.Stack([gate, up, down], [u, u, yug], [yug[h:], yug[:h], yd], wait_prev=[True, False, True],
                   silu_gate=[False, False, True])
    for _ in range(2):
        st.launch()
    torch.cuda.synchronize()
    a, g = up.forward(u), gate.forward(u)
    want = down.forward(a * (g / (1 + torch.exp(-g))))
    assert torch.allclose(yug[:h], a, rtol=1e-6, atol=1e-6) and torch.allclose(yug[h:], g, rtol=1e-6, atol=1e-6)
    assert (yd - want).abs().max() <= 1e-5 * want.abs().max()
    with pytest.raises(rsp.UsageError):  # the gated input is formed in fp32 only
        ub = u.to(torch.bfloat16)
        rsp.Stack([gate, up, down], [ub, ub, yug.to(torch.bfloat16)], [yug[h:], yug[:h], yd],
                  wait_prev=[True, False, True], silu_gate=[False, False, True])
