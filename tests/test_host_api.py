"""Host-side pieces of the reference-named API that need no GPU: weight /
config parsing, the IRLS and non-negativity weight helpers, the chroma
projections of the dense phase (test_energy.py:122-132, 269-282, 363-371)."""
import numpy as np


def test_weights_config_parsing(tmp_path):
    """test_energy.py:363-371."""
    from paper_1908_01961_b200.energy import EnergyWeights, parse_keyvalue_file
    cfg = tmp_path / "weights.cfg"
    cfg.write_text("lambda_data = 100\n# comment\np=0.8\nchroma_reg=identity\n")
    w = EnergyWeights().with_overrides(parse_keyvalue_file(cfg))
    assert w.lambda_data == 100.0
    assert w.p == 0.8
    assert w.chroma_reg == "identity"
    assert w.lambda_clustering == 200.0


def test_solve_config_overrides_types(tmp_path):
    """SolveConfig.with_overrides: floats, booleans and integers from strings;
    unknown keys ignored."""
    from paper_1908_01961_b200.energy import parse_keyvalue_file
    from paper_1908_01961_b200.solver import SolveConfig
    cfg = tmp_path / "solve.cfg"
    cfg.write_text("tol_rel = 1e-3\nrefine = false\npcg_iterations = 8\nunknown = 1\n")
    c = SolveConfig().with_overrides(parse_keyvalue_file(cfg))
    assert c.tol_rel == 1e-3 and c.refine is False and c.pcg_iterations == 8


def test_irls_weight_values():
    """test_energy.py:122-125."""
    from paper_1908_01961_b200.energy import irls_weight
    assert np.isclose(irls_weight(np.array(0.5), 1.0, 1e-3), 2.0)
    assert np.isclose(irls_weight(np.array(0.0), 1.0, 1e-3), 1000.0)
    assert np.isclose(irls_weight(np.array(0.25), 1.0, 1e-3), 4.0)


def test_nonneg_weight_values():
    """test_energy.py:128-132: the boundary T = 0 is penalised."""
    from paper_1908_01961_b200.energy import nonneg_weight
    assert np.isclose(nonneg_weight(np.array(-0.098), 0.002), 10.0)
    assert np.isclose(nonneg_weight(np.array(0.0), 0.002), 500.0)
    assert nonneg_weight(np.array(0.5), 0.002) == 0.0


def test_refine_projection_kills_parallel_updates():
    """test_energy.py:269-282."""
    from paper_1908_01961_b200.energy import chroma_projections
    from paper_1908_01961_b200.palette import BaseColorPalette
    pal = BaseColorPalette(colors=np.array([[0.2, 0.4, 0.6]]))
    P = chroma_projections(pal, "projection")[0]
    b = pal.colors[0]
    assert np.allclose(P @ b, 0.0, atol=1e-12)
    perp = np.array([b[1], -b[0], 0.0])
    assert np.allclose(P @ perp, perp, atol=1e-12)
    assert np.allclose(chroma_projections(pal, "identity")[0], np.eye(3))
