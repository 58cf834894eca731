"""Offline factor build: component scores, component
selection and the sqrt(sigma) split (scores.cpp:15-85, layer.cpp:35-72).

CPU tests pin the reference shim (oracle/_ref) against a numpy restatement;
GPU tests compare csrc/rsp_offline.cu, through the C ABI, with the reference
itself on the same SVD -- bit for bit."""
import numpy as np
import pytest

RNG = np.random.default_rng(2024)


def _case(m=24, n=40, T=5, seed=0):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((m, n))
    u, s, vt = np.linalg.svd(w, full_matrices=False)
    tokens = rng.standard_normal((T, n)) * np.exp(rng.standard_normal(n))
    return w, u, s, vt, tokens


def _np_scores(tokens, s, vt):
    # scores.cpp:15-62, restated: mean over tokens of |sigma_i x_j Vt_ij|
    return np.mean(np.abs(s[:, None, None] * tokens.T[None, :, :] * vt[:, :, None]), axis=2)


def _np_select(scores, r):
    mass = scores.sum(axis=1)
    order = sorted(range(len(mass)), key=lambda i: (-abs(mass[i]), i))
    return np.array(sorted(order[:r]), dtype=np.int64)


def test_ref_scores_and_selection_match_restatement(reforacle):
    w, u, s, vt, tok = _case()
    got = reforacle.aggregate_scores(tok, s, vt)
    np.testing.assert_allclose(got, _np_scores(tok, s, vt), rtol=1e-13, atol=0)
    # the worker count never changes the reference's tree
    assert np.array_equal(reforacle.aggregate_scores(tok, s, vt, workers=4), got)
    for r in (0, 1, 7, 24):
        assert np.array_equal(reforacle.select_components(got, r), _np_select(got, r))


def test_ref_select_ties_and_errors(reforacle):
    sc = np.ones((6, 3))
    sc[4] = 2.0
    assert reforacle.select_components(sc, 3).tolist() == [0, 1, 4]  # ties -> lower index
    from oracle.oracle import UsageError
    with pytest.raises(UsageError):
        reforacle.select_components(sc, 7)
    with pytest.raises(UsageError):
        reforacle.aggregate_scores(np.zeros((0, 3)), np.ones(6), np.ones((6, 3)))


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("T", [1, 5, 16, 33])
def test_gpu_scores_bit_exact(reforacle, cuda, T):
    import torch
    from paper_2504_19449_b200 import offline as off
    w, u, s, vt, tok = _case(m=48, n=72, T=T, seed=T)
    svd = off.SvdResult(torch.from_numpy(u).to(cuda), torch.from_numpy(s).to(cuda), torch.from_numpy(vt).to(cuda))
    got = off.aggregate_scores(list(tok), svd).values.cpu().numpy()
    assert np.array_equal(got, reforacle.aggregate_scores(tok, s, vt))


@pytest.mark.gpu
@pytest.mark.parametrize("r", [0, 1, 5, 24, 48])
def test_gpu_select_components_exact(reforacle, cuda, r):
    import torch
    from paper_2504_19449_b200 import offline as off
    w, u, s, vt, tok = _case(m=48, n=72, T=7, seed=r)
    sc = reforacle.aggregate_scores(tok, s, vt)
    sc[3] = sc[10]  # a tie in row mass
    got = off.select_components(off.ScoreMatrix(torch.from_numpy(sc).to(cuda), 7), r)
    assert got == reforacle.select_components(sc, r).tolist()


@pytest.mark.gpu
def test_gpu_select_components_large_and_ties(cuda):
    import torch
    from paper_2504_19449_b200 import offline as off
    kc, n = 3000, 5  # several chunks of the one-CTA selector
    sc = np.repeat(RNG.integers(0, 50, size=(kc, 1)).astype(np.float64), n, axis=1)
    for r in (1, 100, 2999, 3000):
        got = off.select_components(off.ScoreMatrix(torch.from_numpy(sc).to(cuda), 1), r)
        assert got == _np_select(sc, r).tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("shape,rank", [((48, 32), 6), ((32, 48), 32), ((40, 40), 0)])
def test_gpu_decompose_with_svd_matches_reference(reforacle, coracle, cuda, shape, rank):
    import torch
    from paper_2504_19449_b200 import SparsityPlan
    from paper_2504_19449_b200 import offline as off
    m, n = shape
    w, u, s, vt, tok = _case(m=m, n=n, T=9, seed=m + rank)
    sc = reforacle.aggregate_scores(tok, s, vt)
    a_ref, b_ref, c_ref = reforacle.decompose_with_svd(w, 0.5, rank, sc, u, s, vt)
    svd = off.SvdResult(*(torch.from_numpy(a).to(cuda) for a in (u, s, vt)))
    scores = off.aggregate_scores(torch.from_numpy(tok).to(cuda), svd)
    comps = off.select_components(scores, rank)
    assert comps == c_ref.tolist()
    a_r, b_r = off._split(svd, comps, m, n)
    assert np.array_equal(a_r.cpu().numpy(), a_ref) and np.array_equal(b_r.cpu().numpy(), b_ref)
    layer = off.decompose_with_svd(torch.from_numpy(w), SparsityPlan(0.5, rank), scores, svd, weight_dtype="f32")
    assert layer.selected_components == c_ref.tolist()
    x = RNG.standard_normal(n).astype(np.float32)
    y = layer.forward(torch.from_numpy(x).to(cuda)).cpu().numpy()
    W, A, B = layer.export()
    want = coracle.forward(np.ascontiguousarray(W.T), A, B, 0.5, x.astype(np.float64))
    assert np.max(np.abs(y - want)) <= 1e-5 * max(np.max(np.abs(want)), 1e-30)


@pytest.mark.gpu
def test_gpu_decompose_cusolver_uniform_matches_reference_jacobi(reforacle, cuda):
    """decompose() with a uniform score keeps the leading components; the
    cuSOLVER factors agree with the reference's Jacobi SVD up to the sign of
    each component (a_r b_r is sign-free)."""
    import torch
    from paper_2504_19449_b200 import SparsityPlan
    from paper_2504_19449_b200 import offline as off
    m, n, r = 20, 14, 4
    w = RNG.standard_normal((m, n))
    layer = off.decompose(torch.from_numpy(w), SparsityPlan(0.5, r), off.uniform_scores(m, n), weight_dtype="f32")
    assert layer.selected_components == list(range(r))
    a_ref, b_ref, c_ref = reforacle.decompose_uniform(w, 0.5, r)
    assert c_ref.tolist() == list(range(r))
    _, A, B = layer.export()
    np.testing.assert_allclose(A @ B, a_ref @ b_ref, atol=1e-5 * np.abs(a_ref @ b_ref).max())


@pytest.mark.gpu
def test_gpu_offline_errors(cuda):
    import torch
    from paper_2504_19449_b200 import SparsityPlan, UsageError
    from paper_2504_19449_b200 import offline as off
    w = torch.randn(8, 6, dtype=torch.float64)
    svd = off.svd(w)
    with pytest.raises(UsageError):
        off.aggregate_scores([], svd)
    with pytest.raises(UsageError):
        off.select_components(off.uniform_scores(8, 6), 7)
    with pytest.raises(UsageError):
        off.decompose_with_svd(w, SparsityPlan(0.5, 7), off.uniform_scores(8, 6), svd)
    with pytest.raises(UsageError):
        off.decompose_with_svd(w, SparsityPlan(0.5, 2), off.uniform_scores(6, 8), svd)
