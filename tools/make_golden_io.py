"""Golden fixture for the frame write-out: runs the
reference's pipeline.write_frame_outputs / write_diagnostics on a tiny
deterministic layer stack (imports /root/reference; run in the build
container) and stores every written file's SHA-256 in
tests/golden/frameio.json together with the inputs."""
import hashlib, json, sys, tempfile
from pathlib import Path
import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from lumisplit.energy import LayerStack                      # noqa: E402
from lumisplit.palette import BaseColorPalette, ClusterMap    # noqa: E402
from lumisplit import pipeline as P                           # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "frameio.json"


def inputs():
    rng = np.random.default_rng(7)
    H, W, K = 9, 11, 3
    colors = rng.uniform(0.1, 0.9, size=(K, 3))
    r = rng.normal(-0.7, 0.4, size=(H, W, 3)).astype(np.float32).astype(np.float64)
    T = rng.uniform(-0.05, 0.9, size=(H, W, K + 1)).astype(np.float32).astype(np.float64)
    ids = rng.integers(1, K + 1, size=(H, W)).astype(np.int32)
    return colors, r, T, ids


def main():
    colors, r, T, ids = inputs()
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        P.write_frame_outputs(d, 3, LayerStack(r=r, T=T), BaseColorPalette(colors=colors),
                              ClusterMap(ids=ids, r_cluster=colors[ids - 1]))
        files = {str(p.relative_to(d)): hashlib.sha256(p.read_bytes()).hexdigest()
                 for p in sorted(d.rglob("*")) if p.is_file()}
    # frame 1 after refinement: the cluster map keeps the pre-refinement
    # palette's reflectance while the layers are written with the refined one
    cluster_colors = np.clip(colors + np.array([0.05, -0.03, 0.02]), 0.0, 1.0)
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        P.write_frame_outputs(d, 1, LayerStack(r=r, T=T), BaseColorPalette(colors=colors),
                              ClusterMap(ids=ids, r_cluster=cluster_colors[ids - 1]))
        files_rc = {str(p.relative_to(d)): hashlib.sha256(p.read_bytes()).hexdigest()
                    for p in sorted(d.rglob("*")) if p.is_file()}
    OUT.write_text(json.dumps({"colors": colors.tolist(), "r": r.tolist(), "T": T.tolist(),
                               "ids": ids.tolist(), "files": files,
                               "cluster_colors": cluster_colors.tolist(),
                               "files_cluster_palette": files_rc}) + "\n")
    print(f"wrote {OUT} ({len(files)} files)")


if __name__ == "__main__":
    main()
