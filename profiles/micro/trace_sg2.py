"""Timeline of one SG2 CTA (developer tool; needs the -DLGD_TRACE build):
   LGD_LIBRARY=build/trace/liblegend_b200.so python profiles/micro/trace_sg2.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2505_09258_b200 as lgd  # noqa: E402

rng = np.random.default_rng(1)
V, d, k, C_, P = 200000, 100, 1000, 1000, 100000
edges = np.stack([rng.integers(0, V, P), rng.integers(0, 16, P), rng.integers(0, V, P)],
                 1).astype(np.uint32)
t = lgd.Trainer(lgd.ScoreModel("distmult", d),
                lgd.TrainOptions(batch_size=P, negatives=k, shared_chunk=C_))
t.set_graph(edges, V, 16)
t.make_partition_plan(1)
t.init_store(1)
shared = rng.integers(0, V, (P // C_) * k).astype(np.uint32)
for _ in range(3):
    t.train_batch(edges, shared)
buf = np.zeros((2, 4096), np.uint64)
lgd.library().lgd_debug_trace(buf.ctypes.data_as(C.c_void_p))
names = {"control": ["start", "S+1 issued", "W seen", "mix issued", "mix done"],
         "warp 1": ["start", "S ready", "W computed", "W free", "W written"]}
for who, row in (("control", buf[0]), ("warp 1", buf[1])):
    t0 = int(row[0])
    print(who)
    for nb in range(16):
        vals = [int(row[nb * 8 + i]) - t0 if row[nb * 8 + i] else -1 for i in range(5)]
        print(f"  block {nb:2d}: " + "  ".join(f"{n}={v}" for n, v in zip(names[who], vals)
                                              if v >= 0))
