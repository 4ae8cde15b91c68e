"""Timing of correct_reflectance's K candidate solves (correction.py:168-201):
one at a time (_candidate_sparsity, the thread-pool layout's GPU schedule)
against the batched launch sequence (_candidate_batch, ls_flip_flop_batch).

python tools/correction_probe.py [H W K box]
A synthetic clip frame (synth.make_clip), segmented with its generator palette;
the region is the flood fill of the cluster at the frame centre clipped to a
box x box window, so its padded bounding box is about (box+32)^2 pixels.
Prints one JSON line.
"""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_01961_b200 import correction as C, synth  # noqa: E402
from paper_1908_01961_b200.energy import EnergyWeights  # noqa: E402
from paper_1908_01961_b200.imaging import Frame  # noqa: E402
from paper_1908_01961_b200.palette import BaseColorPalette, segment  # noqa: E402
from paper_1908_01961_b200.solver import SolveConfig  # noqa: E402


def main():
    H, W, K, box = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1080, 1920, 8, 192)))
    dev = torch.device("cuda", 0)
    clip = synth.make_clip(H, W, K, 1, seed=0, device=dev)
    pal = BaseColorPalette(colors=clip.colors)
    frame = Frame(clip.frames[0])
    cmap = segment(frame, pal)
    cy, cx = H // 2, W // 2
    region = C.identify_region((cx, cy), cmap, frame=frame)
    win = torch.zeros_like(region.mask)
    win[max(0, cy - box // 2):cy + box // 2, max(0, cx - box // 2):cx + box // 2] = True
    region.mask &= win
    y0, y1, x0, x1 = region.bbox(C.BBOX_PAD)
    cfg = SolveConfig(outer_iterations=8, refine=False)
    w = EnergyWeights()
    ks = list(range(1, K + 1))

    def seq():
        return [C._candidate_sparsity(frame, cmap, pal, region, k, w, cfg, 0) for k in ks]

    def bat():
        b = C._candidate_batch(frame, cmap, pal, region, ks, w, cfg, 0)
        return [b[k] for k in ks]

    out = {"H": H, "W": W, "K": K, "region_px": region.size, "bbox": [y1 - y0, x1 - x0]}
    for name, fn in (("sequential", seq), ("batched", bat)):
        fn()                                  # warm (contexts, graphs)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            scores = fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[name + "_ms"] = min(ts)
        out[name + "_scores"] = scores
    out["bitwise_equal"] = out["sequential_scores"] == out["batched_scores"]
    out["pick"] = C.correct_reflectance(region, frame, cmap, pal, config=cfg)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
