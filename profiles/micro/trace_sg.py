"""Timelines of one CTA of SG1 / SG2 / SG3 (developer tool; needs the -DLGD_TRACE
build, e.g. make -C paper_2505_09258_b200/csrc OUT=$PWD/paper_2505_09258_b200/trace/liblegend_b200.so
OBJDIR=$PWD/build/obj_trace NVFLAGS_EXTRA=-DLGD_TRACE):
   LGD_LIBRARY=paper_2505_09258_b200/trace/liblegend_b200.so python profiles/micro/trace_sg.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2505_09258_b200 as lgd  # noqa: E402

rng = np.random.default_rng(1)
V, d, k, C_, P = 2000000, 100, 1000, 1000, 100000
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
buf = np.zeros((3, 2, 4096), np.uint64)
lgd.library().lgd_debug_trace(buf.ctypes.data_as(C.c_void_p))
names = {
    0: {"control": ["top", "S+1 issued", "S done"], "warp 1": ["top", "S ready", "stats done"]},
    1: {"control": ["top", "S+1 issued", "S done", "W seen", "mix issued", "mix done"],
        "warp 1": ["top", "S ready", "W computed", "W free", "W written"]},
    2: {"control": ["top", "S+1 issued", "S done", "W seen", "IR1T landed", "G done"],
        "warp 1": ["top", "S ready", "W computed", "W free", "W written"]},
}
for kid, kname in enumerate(["SG1", "SG2", "SG3"]):
    if not buf[kid].any():
        continue
    print(f"===== {kname}")
    for w, who in enumerate(("control", "warp 1")):
        row = buf[kid, w]
        t0 = int(row[4090]) if row[4090] else int(row[row > 0].min())
        print(f"  {who}: kernel body {int(row[4091]) - t0 if row[4091] else -1} cycles;"
              f" marks 4000={int(row[4000]) - t0 if row[4000] else -1}"
              f" 4001={int(row[4001]) - t0 if row[4001] else -1}"
              f" 4010={int(row[4010]) - t0 if row[4010] else -1}")
        print("    tail marks: " + " ".join(f"{m}={int(row[m]) - t0}" for m in range(4001, 4010)
                                          if row[m]))
        for nb in range(10):
            vals = [int(row[nb * 8 + i]) - t0 if row[nb * 8 + i] else -1
                    for i in range(len(names[kid][who]))]
            if all(v < 0 for v in vals):
                continue
            print(f"    block {nb:2d}: " + "  ".join(f"{n}={v}" for n, v in
                                                    zip(names[kid][who], vals) if v >= 0))
