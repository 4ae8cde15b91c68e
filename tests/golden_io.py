"""Load golden fixtures (tests/golden/*.npz, made by tools/make_golden.py
from the reference) into oracle objects."""
from pathlib import Path

import numpy as np

from oracle import lumisplit_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def oracle_aux(d):
    pairs = O.Pairs(src=d["pair_src"], dst=d["pair_dst"], temporal=d["pair_temporal"],
                    weight=d["pair_weight"], shape=d["image"].shape[:2])
    return O.Aux(edge=d["edge"], pairs=pairs, prev_r=d.get("prev_r"),
                 cluster_ids=d.get("cluster_ids"), r_cluster_log=d.get("r_cluster_log"))


def oracle_system(d):
    return O.FrozenSystem(d["image"], d["colors"], d["r0"], d["T0"], oracle_aux(d), O.Weights())


def records_array(records):
    rows = []
    for rec in records:
        pc = rec.get("pcg", {"iterations": -1, "initial_residual": np.nan,
                             "final_residual": np.nan})
        rows.append([0.0 if rec["phase"] == "sparse" else 1.0, rec["energy_before"],
                     rec["energy_after"], float(rec["accepted"]), rec["alpha"],
                     pc["iterations"], pc["initial_residual"], pc["final_residual"],
                     rec.get("delta_b_norm", np.nan)])
    return np.array(rows)
