"""Golden fixtures for the correction and editing rows (SURVEY.md 8(f) item
4), from the reference itself (imports /root/reference; build container):
  tests/golden/correction.npz -- flood fills (identify / merge / track) on a
      synthetic id map, and correct_reflectance's pick on a synthetic frame
      whose region was relabelled to a wrong cluster;
  tests/golden/editing.npz -- recolor / suppress_spill / rekey_background."""
import sys
from pathlib import Path
import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lumisplit import correction as RC, editing as RE        # noqa: E402
from lumisplit.energy import LayerStack                        # noqa: E402
from lumisplit.imaging import Frame                            # noqa: E402
from lumisplit.palette import BaseColorPalette, ClusterMap, segment   # noqa: E402
from lumisplit.solver import SolveConfig                       # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def flood_cases():
    rng = np.random.default_rng(3)
    H, W, K = 37, 45, 3
    ids = rng.integers(1, K + 1, size=(H, W)).astype(np.int32)
    ids[5:20, 8:30] = 2                     # a big connected blob
    ids[25:33, 2:40] = 3
    cmap = ClusterMap(ids=ids, r_cluster=np.zeros((H, W, 3)))
    r1 = RC.identify_region((10, 10), cmap)
    r2 = RC.identify_region((20, 28), cmap, merge_into=None)
    ids2 = ids.copy()
    ids2[10:15, 8:30] = 1                   # the next frame cuts the blob
    track = RC.track_region(r1, ClusterMap(ids=ids2, r_cluster=np.zeros((H, W, 3))), frame_index=1)
    return {"ids": ids, "ids2": ids2, "m_identify": r1.mask, "m_identify2": r2.mask,
            "m_track": track.mask, "src1": r1.source_id, "src2": r2.source_id}


def correction_case():
    from paper_1908_01961_b200 import synth
    clip = synth.make_clip(48, 64, 3, 1, seed=5, device="cpu")
    img = clip.frames[0].double().numpy()
    colors = np.asarray(clip.colors, dtype=np.float64)
    pal = BaseColorPalette(colors=colors)
    cmap = segment(Frame(img), pal)
    ids = cmap.ids.copy()
    # relabel the biggest connected piece of cluster 2 to the wrong cluster 3
    true_id, wrong_id = 2, 3
    ys, xs = np.nonzero(ids == true_id)
    y, x = int(ys[len(ys) // 2]), int(xs[len(xs) // 2])
    seed = np.zeros_like(ids, dtype=bool)
    seed[y, x] = True
    blob = RC._flood(ids, seed, true_id)
    ids[blob] = wrong_id
    bad = ClusterMap(ids=ids, r_cluster=colors[ids - 1])
    region = RC.identify_region((x, y), bad, frame=Frame(img))
    cfg = SolveConfig(outer_iterations=4, refine=False)
    pick = RC.correct_reflectance(region, Frame(img), bad, pal, config=cfg, max_workers=1)
    from lumisplit.energy import EnergyWeights
    scores = [RC._candidate_sparsity(Frame(img), bad, pal, region, k, EnergyWeights(), cfg, 0)
              for k in range(1, 4)]
    return {"c_image": img.astype(np.float32), "c_colors": colors, "c_ids": ids, "c_click": np.array([x, y]),
            "c_mask": region.mask, "c_pick": pick, "c_true": true_id, "c_outer": 4,
            "c_scores": np.array(scores)}


def editing_case():
    rng = np.random.default_rng(11)
    H, W, K = 10, 12, 3
    colors = rng.uniform(0.1, 0.9, size=(K, 3))
    r = rng.normal(-0.6, 0.3, size=(H, W, 3)).astype(np.float32).astype(np.float64)
    T = rng.uniform(0.0, 0.8, size=(H, W, K + 1)).astype(np.float32).astype(np.float64)
    ids = rng.integers(1, K + 1, size=(H, W)).astype(np.int32)
    pal = BaseColorPalette(colors=colors)
    cmap = ClusterMap(ids=ids, r_cluster=colors[ids - 1])
    L = LayerStack(r=r, T=T)
    bg = rng.uniform(0.0, 1.0, size=(H, W, 3)).astype(np.float32).astype(np.float64)
    matte = rng.uniform(size=(H, W)) < 0.3
    new = np.array([0.2, 0.7, 0.4])
    return {"e_colors": colors, "e_r": r, "e_T": T, "e_ids": ids, "e_bg": bg, "e_matte": matte, "e_new": new,
            "e_recolor": RE.recolor(L, pal, 2, new, cmap), "e_spill": RE.suppress_spill(L, pal, 3),
            "e_rekey": RE.rekey_background(L, pal, 1, Frame(bg), matte)}


if __name__ == "__main__":
    out = ROOT / "tests" / "golden"
    np.savez_compressed(out / "correction.npz", **flood_cases(), **correction_case())
    np.savez_compressed(out / "editing.npz", **editing_case())
    d = np.load(out / "correction.npz")
    print("pick", d["c_pick"], "true", d["c_true"], "mask px", d["c_mask"].sum(), "scores", d["c_scores"])
