"""Per-rank compute of the column-sharded reduction H = L^-1 A L^-H at c4 scale, timed
rank by rank on ONE GPU (no collective; the shards are independent): shows the
balance of distributed.reduction_bounds and the per-rank time an N-GPU run would see
before its all-gather.

    python scripts/reduce_shard_probe.py [n] > gpurun_out/reduce_shard.json
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402
from paper_1305_5120_b200.distributed import ColumnShards, reduction_bounds  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
g = torch.Generator(device=dev)
g.manual_seed(0)
a = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
linv = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g).tril_()
linv = linv.transpose(0, 1).contiguous()  # (cols, rows) block of a lower-triangular matrix
out = {"n": n}
for world in (1, 2, 4, 8):
    sh = ColumnShards(n, world, reduction_bounds(n, world))
    times = []
    for rank in range(world):
        lo, hi = sh.range(rank)
        w = hi - lo
        x = D.empty(n, w, dev)
        hp = D.empty(n, w, dev)
        for rep in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.zgemm("N", "C", n, w, n, 1.0, a, linv[:, lo:hi], 0.0, x,
                      tri=eng.TRI_B_UPPER, tri_offset=lo)
            eng.zgemm("N", "N", n, w, n, 1.0, linv, x, 0.0, hp, tri=eng.TRI_A_LOWER)
            e1.record()
            torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        del x, hp
    out[str(world)] = {"bounds": sh.bounds, "rank_s": times, "max_s": max(times),
                       "tflops_per_gpu_at_max": 8.0 * n ** 3 / max(times) / world / 1e12}
    print(world, [round(t, 3) for t in times], flush=True)
print(json.dumps(out))
