#!/usr/bin/env python
"""Permute bandwidth of the shapes the config-5 planner permutes (sweep
instances with interleaved contracted / free legs): candidate target orders."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402

CASES = [  # (dtype, shape, perm)
    ("r64", (3, 8, 8, 37, 5, 37), (0, 2, 4, 1, 3, 5)),      # small: OMxuHR -> O x H M u R
    ("r64", (3, 8, 8, 37, 5, 37), (0, 2, 4, 5, 3, 1)),      # small: OMxuHR -> O x H R u M
    ("r64", (37, 64, 37, 8), (1, 0, 2, 3)),                 # small: RduM -> d R u M
    ("r64", (37, 64, 37, 8), (1, 3, 2, 0)),                 # small: RduM -> d M u R
    ("r32", (37, 8, 128, 7, 7, 128), (1, 2, 3, 5, 0, 4)),   # rXcByH -> X c B H r y
    ("r32", (37, 8, 128, 7, 7, 128), (0, 4, 1, 2, 3, 5)),   # rXcByH -> r y X c B H
    ("r32", (7, 64, 7, 64, 256, 5), (0, 1, 2, 4, 5, 3)),    # xdKTQF -> x d K Q F T
    ("r32", (7, 64, 7, 64, 256, 5), (3, 0, 1, 2, 4, 5)),    # xdKTQF -> T x d K Q F
    ("r64", (7, 32, 16, 1, 5, 16, 32, 3, 7), (0, 1, 2, 3, 4, 5, 6, 7, 8)),
]


def main():
    ctx = tci.Context(0)
    out = []
    for dt, shape, perm in CASES:
        x = synth.random_tensor(shape, dt, 3, 1, device="cuda")
        y = torch.empty([shape[p] for p in perm], dtype=x.dtype, device="cuda")
        for _ in range(2):
            ctx.permute(x, list(perm), out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ctx.permute(x, list(perm), out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        r = {"dtype": dt, "shape": shape, "perm": perm, "ms": ms,
             "TBs": 2 * x.numel() * x.element_size() / ms / 1e9}
        print(json.dumps(r), flush=True)
        out.append(r)
        del x, y
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "permute_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
