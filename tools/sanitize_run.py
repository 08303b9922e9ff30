"""A small run through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): the R <= 16 MTTKRP, the lean MTTKRP at R pitch 64 (x broadcast) and 256, the DMMA
row updates (R <= 64 and R > 64), the DMMA Gram, the FMA kernels (fp32), the snapshot and
Jacobi variants, emulated ranks with the delta exchange, predict / RMSE.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2003_03572_b200.sacd import Sacd  # noqa: E402


def tensor(dims, nnz, seed):
    rng = np.random.default_rng(seed)
    key = np.unique(rng.integers(0, dims[0] * dims[1] * dims[2], size=nnz * 2))[:nnz]
    rng.shuffle(key)
    c = np.stack([key // (dims[1] * dims[2]), (key // dims[2]) % dims[1], key % dims[2]], 1).astype(np.uint32)
    c[: nnz // 10, 0] = 1  # a heavy slice: split rows and fix-ups
    key = np.unique(c[:, 0].astype(np.int64) * dims[1] * dims[2] + c[:, 1].astype(np.int64) * dims[2] + c[:, 2])
    c = np.stack([key // (dims[1] * dims[2]), (key // dims[2]) % dims[1], key % dims[2]], 1).astype(np.uint32)
    v = (rng.random(len(key)) + 0.5).astype(np.float32)
    return c, v


dims = (120, 90, 70)
c, v = tensor(dims, 6000, 1)
cases = [dict(rank=5), dict(rank=40), dict(rank=200), dict(rank=40, precision="f32"),
         dict(rank=40, variant="snapshot"), dict(rank=12, variant="jacobi"),
         dict(rank=40, emulate_ranks=3, exchange="delta"), dict(rank=40, nnz_per_item=64)]
for kw in cases:
    R = kw.pop("rank")
    with Sacd(c, v, dims, R, 3, **kw) as g:
        g.iterate(3)
        f, fit = g.fit()
        g.factors()
        r = g.rmse(c[:500], v[:500])
        print(f"R={R} {kw}: f={f:.6e} rmse={r:.4f}", flush=True)
print("sanitize run done")
