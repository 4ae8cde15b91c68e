"""Seeds whose PCG64 u32 stream has a zero word (a Lemire rejection of the
range-15 partner draws, energy.py:163-169) among the first 8 N words -- the
dx / dy sections of an H x W frame's consistency sampling.  Used to pick the
seed of tests/test_gpu_scale.py's rejection case.

python tools/find_rejection_seed.py [H W n_seeds]
"""
import sys

import numpy as np


def zeros(seed: int, n_words: int) -> np.ndarray:
    raw = np.random.PCG64(seed).random_raw((n_words + 1) // 2)
    u32 = raw.view(np.uint32)[:n_words]        # low half first (little-endian)
    return np.nonzero(u32 == 0)[0]


def main():
    H, W, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (1080, 1920, 600)))
    N = H * W
    for seed in range(n):
        z = zeros(seed, 8 * N)
        if z.size:
            print(seed, z.tolist(), flush=True)


if __name__ == "__main__":
    main()
