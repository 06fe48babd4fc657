import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import bench, paper_2505_09258_b200 as lgd
cfg = bench.CONFIGS["tw"]
t = bench.setup_trainer(cfg, 0)
host = lgd.PinnedArray((t.num_edges, 3), np.uint32)
t.bucketed_edges(host.array)
for g in range(3, 11):
    t0 = time.perf_counter()
    r = t.train_buckets_from_host(1, g, g + 1, host.array)
    w = time.perf_counter() - t0
    print(g, f"wall {w*1e3:.1f} ms  device {r.device_ms:.1f} ms  edges {r.edges_trained}  h2d {r.h2d_bytes/1e6:.1f} MB")
