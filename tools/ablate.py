"""Timing ablations of k_pcg_apply: builds liblumisplit_b200 variants with
-DLS_ABLATE=n into tools/_ablate/ (1: no consistency term, 2: no p formation,
3: no smoothness, 4: no r-sparsity; n+100: the same with 4 CTAs/SM; 201: 2 CTAs/SM via a
shared-memory pad; 202: the x-update loads issued before the stage barrier) and, with --run, times each through
bench.py --profile-only.  Results are wrong by construction; timing only."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1908_01961_b200 import build as B

OUT = ROOT / "tools" / "_ablate"

def build_variant(n, extra=()):
    OUT.mkdir(exist_ok=True)
    objs = []
    procs = []
    for src in B.SRC:
        obj = OUT / f"{src.stem}_{n}.o"
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, f"-DLS_ABLATE={n % 100 if n < 200 else 0}", *extra, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        procs.append(subprocess.Popen(cmd)); objs.append(str(obj))
    assert all(p.wait() == 0 for p in procs)
    so = OUT / f"lib_{n}.so"
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC", *objs, "-o", str(so)])
    return so

if __name__ == "__main__":
    variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 and sys.argv[1] != "--run" else [1, 2, 3, 4]
    if "--run" not in sys.argv:
        for n in variants:
            extra = []
            if 100 <= n < 200:
                extra = ["-DLS_PCG_MINB=4"]
            elif n == 201:      # occupancy pinned to 2 CTAs / SM (smem pad)
                extra = ["-DLS_PCG_PAD=30000"]
            elif n == 202:      # x-update loads issued before the stage barrier
                extra = ["-DLS_XEARLY=1"]
            elif n == 204:      # x-update fma/stores deferred past the next tile's operand wait
                extra = ["-DLS_XDEFER=1"]
            elif n == 205:      # energy kernel at 2 CTAs/SM (more registers, no rematerialisation)
                extra = ["-DLS_EG_MINB=2"]
            elif n == 206:      # sampler: 4 pixels per thread (now the default)
                extra = ["-DLS_SAMPLE_PIX=4"]
            elif n == 207:      # operator: the p window loaded with the tile's other windows (round 1)
                extra = ["-DLS_PEARLY=0"]
            elif n == 208:      # operator: p_{i-1} read from L2 in the formation, 4 CTAs/SM (64 registers)
                extra = ["-DLS_PFORM_GLOBAL=1", "-DLS_PCG_MINB=4"]
            elif n == 209:      # operator: p_{i-1} read from L2 in the formation, 3 CTAs/SM
                extra = ["-DLS_PFORM_GLOBAL=1"]
            elif n == 210:      # tile coordinates by div / mod every tile (before the incremental walk)
                extra = ["-DLS_TILEWALK=0"]
            elif n == 212:      # sampler: 2 pixels per thread
                extra = ["-DLS_SAMPLE_PIX=2"]
            elif n == 213:      # sampler: 8 pixels per thread (the round-2 default before 4)
                extra = ["-DLS_SAMPLE_PIX=8"]
            elif n == 211:      # update: a float4's products summed in fp32 before the fp64 accumulators
                extra = ["-DLS_UPD_F32P=1"]
            build_variant(n, extra)
    else:
        for n in [0] + variants:
            env = dict(os.environ)
            if n:
                env["LS_LIB_PATH"] = str(OUT / f"lib_{n}.so")
            r = subprocess.run([sys.executable, "bench.py", "--profile-only", "--steps", "5", "--warmup", "3"],
                               env=env, capture_output=True, text=True, cwd=ROOT)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                pk = d["roofline"]["per_kernel"]
                print(n, {k: round(v["avg_us"], 1) for k, v in pk.items()},
                      {"fps": round(d["value"], 2), "ms_per_frame": round(d["ms_per_step"], 3)}, flush=True)
            except Exception as e:
                print(n, "failed", r.stderr[-800:], flush=True)
