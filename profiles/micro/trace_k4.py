"""Per-piece timeline of a few K4 warps (developer tool; -DLGD_TRACE build):
   LGD_LIBRARY=build/trace/liblegend_b200.so python profiles/micro/trace_k4.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2505_09258_b200 as lgd  # noqa: E402

t = bench.setup_trainer(bench.CONFIGS["tw"], 0)
t.train_buckets(0, 0, 2)
buf = np.zeros((8, 1024), np.uint64)
lgd.library().lgd_debug_trace_k4(buf.ctypes.data_as(C.c_void_p))  # reset
t.train_buckets(0, 2, 3)
lgd.library().lgd_debug_trace_k4(buf.ctypes.data_as(C.c_void_p))
names = {1: "top", 2: "staged", 3: "item0", 4: "items", 5: "adagrad"}
for w in range(3):
    ev = [(int(buf[w, 2 * i]), int(buf[w, 2 * i + 1])) for i in range(512) if buf[w, 2 * i]]
    if not ev:
        continue
    print(f"warp sample {w}: {len(ev)} events")
    t0 = ev[0][0]
    prev = t0
    line = []
    for c, tag in ev[:120]:
        base = tag if tag < 16 else 2
        extra = f"(n={tag // 16})" if tag >= 16 else ""
        line.append(f"{names.get(base, base)}{extra}+{c - prev}")
        prev = c
        if base == 1 and len(line) > 1:
            print("   ", " ".join(line[:-1]))
            line = line[-1:]
