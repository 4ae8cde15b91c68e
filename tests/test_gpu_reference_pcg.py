"""The reference's PCG / Gauss-Newton solver tests (test_solver.py:24-37,
54-69, 135-186) pointed at the sm_100a path.

The reference checks its fp64 PCG against a dense direct solve of the
explicitly materialised normal matrix.  Here the explicit matrix and the
direct solve come from the CPU oracle (fp64, pinned to the reference by
tests/test_oracle_golden.py) on the same problem, and the device solver (fp32
vectors, fp64 reductions) is held to the reference's own tolerances where
fp32 allows it (rel < 1e-3 for PCG(16) on 2x2 problems) and to 1e-4 for the
full-budget solve (the reference asks 1e-6 of fp64; fp32 vectors carry ~1e-7
per operation and the 20-step recurrence amplifies that by the condition
number).
"""
import numpy as np
import pytest
import torch

from oracle import lumisplit_oracle as O
from tests.golden_io import load

COLORS = ([[0.80, 0.15, 0.10]], [[0.10, 0.75, 0.15]], [[0.15, 0.2, 0.8]])


# ---------------------------------------------------------------------------
# host PCG (solver.pcg is the reference-named generic routine; CPU only)
# ---------------------------------------------------------------------------

def test_pcg_zero_rhs_returns_zero():
    """test_solver.py:24-28."""
    from paper_1908_01961_b200.solver import pcg
    x, info = pcg(lambda v: v, np.zeros(5), np.ones(5), 16)
    assert np.all(np.asarray(x) == 0)
    assert info["iterations"] == 0


def test_pcg_solves_spd_system():
    """test_solver.py:31-37."""
    from paper_1908_01961_b200.solver import pcg
    rng = np.random.default_rng(0)
    M = rng.normal(size=(12, 12))
    A = M @ M.T + 12 * np.eye(12)
    b = rng.normal(size=12)
    x, _ = pcg(lambda v: A @ v, b, np.diag(A), 16)
    assert np.linalg.norm(A @ np.asarray(x) - b) < 1e-8 * np.linalg.norm(b)


# ---------------------------------------------------------------------------
# device solver
# ---------------------------------------------------------------------------

def _small_problem(seed, h, w, colors):
    """A tiny problem with every term active and IRLS weights in a sane range
    (log-reflectance ramp, ~12% negative layer values to switch the
    non-negativity term on), the recipe of test_solver.py:103-132."""
    rng = np.random.default_rng(seed)
    colors = np.asarray(colors, dtype=np.float64)
    K = colors.shape[0]
    yy, xx = np.mgrid[0:h, 0:w]
    ramp = (xx + yy) / max(h + w, 1)
    r = np.minimum(np.log(0.4) + 0.1 * ramp[:, :, None] + 0.02 * rng.uniform(size=(h, w, 3)), 0.0)
    T = 0.5 + 0.1 * ramp[:, :, None] + 0.03 * rng.uniform(size=(h, w, K + 1))
    neg = rng.uniform(size=(h, w, K + 1)) < 0.12
    T[neg] = -rng.uniform(0.08, 0.2, size=int(neg.sum()))
    B = O.palette_matrix(colors)
    image = np.clip(np.exp(r) * np.tensordot(np.abs(T), B, axes=([2], [0]))
                    * rng.uniform(0.95, 1.05, size=(h, w, 1)), 0.02, 1.0)
    inten = image.sum(axis=2)
    chroma = image[:, :, :2] / inten[:, :, None]
    anchor = np.log(np.maximum(np.exp(r) * rng.uniform(0.95, 1.05, size=(h, w, 3)), O.LOG_FLOOR))
    # everything the device sees is fp32: round once and give the oracle the same values
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    image, r, T, anchor = f32(image), f32(r), f32(T), f32(anchor)
    edge = f32(O.edge_gate(chroma))
    pairs = O.sample_pairs(chroma, None, seed + 1)
    return dict(image=image, colors=colors, r0=r, T0=T, edge=edge, r_cluster_log=anchor,
                pair_src=pairs.src, pair_dst=pairs.dst, pair_temporal=pairs.temporal,
                pair_weight=pairs.weight)


def _oracle(d):
    pairs = O.Pairs(src=d["pair_src"], dst=d["pair_dst"], temporal=d["pair_temporal"],
                    weight=d["pair_weight"], shape=d["image"].shape[:2])
    aux = O.Aux(edge=d["edge"], pairs=pairs, r_cluster_log=d["r_cluster_log"])
    return O.FrozenSystem(d["image"], d["colors"], d["r0"], d["T0"], aux, O.Weights())


def _device(d):
    from paper_1908_01961_b200.energy import (ConsistencySamples, EnergyAux, EnergyWeights,
                                              LayerStack, assemble_blocks)
    from paper_1908_01961_b200.palette import BaseColorPalette
    t = lambda a, dt=torch.float32: torch.as_tensor(np.asarray(a), dtype=dt, device="cuda")  # noqa: E731
    samples = ConsistencySamples(src=t(d["pair_src"], torch.int64), dst=t(d["pair_dst"], torch.int64),
                                 temporal=t(d["pair_temporal"], torch.bool),
                                 weight=t(d["pair_weight"], torch.float64), shape=d["image"].shape[:2])
    aux = EnergyAux(edge_weights=t(d["edge"]), samples=samples, r_cluster_log=t(d["r_cluster_log"]))
    # a raw (H, W, 3) array, as the reference's small_problem passes (no Frame size check)
    return assemble_blocks(t(d["image"]), BaseColorPalette(colors=d["colors"]),
                           LayerStack(t(d["r0"]), t(d["T0"])), aux, EnergyWeights())


def _explicit(osys, n):
    return np.stack([osys.apply(np.eye(n)[j]) for j in range(n)], axis=1)


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(len(COLORS)))
def test_pcg16_matches_direct_solve_small_problems(ci):
    """test_solver.py:135-153: on 2x2 problems the 16-step budget converges,
    so the device PCG(16) step ties out with a dense direct solve."""
    from paper_1908_01961_b200.energy import to_reference_vector
    for seed in range(5):
        d = _small_problem(seed, 2, 2, COLORS[ci])
        osys = _oracle(d)
        b, diag = osys.grad_diag()
        A = _explicit(osys, b.size)
        assert np.allclose(A, A.T, rtol=0, atol=1e-9 * np.abs(A).max())
        direct = np.linalg.solve(A, b)
        blocks = _device(d)
        db, ddiag = blocks.gradient_and_diag()
        assert np.max(np.abs(to_reference_vector(db).cpu().numpy() - b)) < 1e-5 * np.abs(b).max()
        assert np.max(np.abs(to_reference_vector(ddiag).cpu().numpy() - np.diag(A))) < 1e-5 * np.abs(A).max()
        x, info = blocks.pcg(16)
        xv = to_reference_vector(x).double().cpu().numpy()
        rel = np.linalg.norm(xv - direct) / np.linalg.norm(direct)
        assert rel < 1e-3, f"colors {COLORS[ci]} seed {seed}: rel diff {rel} ({info})"


@pytest.mark.gpu
def test_device_operator_columns_equal_explicit_normal_matrix():
    """test_solver.py:40-51 on the device: the fused J^T J applied to every
    unit vector reproduces the explicitly materialised normal matrix."""
    from paper_1908_01961_b200.energy import from_reference_vector, to_reference_vector
    d = _small_problem(7, 3, 4, [[0.6, 0.3, 0.1], [0.2, 0.3, 0.7]])
    osys = _oracle(d)
    n = osys.grad_diag()[0].size
    A = _explicit(osys, n)
    blocks = _device(d)
    H, W = d["image"].shape[:2]
    K = d["colors"].shape[0]
    cols = []
    for j in range(n):
        e = from_reference_vector(np.eye(n)[j], H, W, K)
        cols.append(to_reference_vector(blocks.apply_normal(e)).double().cpu().numpy())
    Ad = np.stack(cols, axis=1)
    assert np.max(np.abs(Ad - A)) < 2e-5 * np.abs(A).max()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ops_a", "ops_b", "ops_c", "ops_d"])
def test_pcg16_residual_reduction_on_8x8(name):
    """test_solver.py:156-177: at 8x8 the 16-step solve is inexact but
    contracts the residual at least tenfold."""
    from tests.test_gpu_parity import device_problem
    from paper_1908_01961_b200.energy import assemble_blocks
    frame, pal, layers, aux, w = device_problem(load(name))
    _, info = assemble_blocks(frame, pal, layers, aux, w).pcg(16)
    assert info["initial_residual"] >= 10.0 * info["final_residual"]


@pytest.mark.gpu
def test_pcg_converges_given_capacity_budget():
    """test_solver.py:180-186: with an n-iteration budget the device PCG
    matches the direct solve (fp32 vectors: 1e-4 instead of fp64's 1e-6)."""
    from paper_1908_01961_b200.energy import to_reference_vector
    d = _small_problem(2, 2, 2, COLORS[0])
    osys = _oracle(d)
    b, _ = osys.grad_diag()
    direct = np.linalg.solve(_explicit(osys, b.size), b)
    x, _ = _device(d).pcg(b.size)
    xv = to_reference_vector(x).double().cpu().numpy()
    assert np.linalg.norm(xv - direct) / np.linalg.norm(direct) < 1e-4


@pytest.mark.gpu
def test_gn_zero_residual_stationary():
    """test_solver.py:54-69: an exactly factorable uniform frame with every
    prior at its optimum is a stationary point (zero right-hand side: PCG
    takes no iteration and the state does not move)."""
    from paper_1908_01961_b200.energy import EnergyWeights, LayerStack
    from paper_1908_01961_b200.imaging import Frame
    from paper_1908_01961_b200.palette import BaseColorPalette, ClusterMap
    from paper_1908_01961_b200.solver import SolveConfig, SolverState, build_aux, gn_step_sparse
    h = w = 8
    frame = Frame(torch.full((h, w, 3), 0.25, device="cuda"))
    pal = BaseColorPalette(colors=np.array([[1.0, 1.0, 1.0]]))
    T = torch.zeros(h, w, 2, device="cuda")
    T[:, :, 0] = 0.25                     # R = 1, T0 = 0.25 reproduces I exactly
    layers = LayerStack(torch.zeros(h, w, 3, device="cuda"), T)
    cm = ClusterMap(ids=torch.ones(h, w, dtype=torch.int32, device="cuda"),
                    r_cluster=torch.ones(h, w, 3, device="cuda"))
    st = SolverState(frame=frame, palette=pal, layers=layers, aux=build_aux(frame, cm, seed=0),
                     weights=EnergyWeights(), config=SolveConfig())
    rec = gn_step_sparse(st)
    assert rec["energy_before"] < 1e-20
    assert rec["pcg"]["iterations"] == 0
    assert torch.allclose(st.layers.T[:, :, 0], torch.full((h, w), 0.25, device="cuda"))
    assert rec["energy_after"] <= rec["energy_before"] + 1e-20
