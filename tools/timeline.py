#!/usr/bin/env python3
"""Per-CTA timeline of one cp.async-engine launch (TCR_DEBUG_MODE=20 %globaltimer stamps):
start spread, streaming-end spread (the tail), last-CTA finalise.  Profiling tool.
    python tools/timeline.py [--n 1073741824] [--R 1] [--B 1024]"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 30)
    ap.add_argument("--R", type=int, default=1)
    ap.add_argument("--B", type=int, default=1024)
    a = ap.parse_args()
    os.environ["TCR_DEBUG_MODE"] = "20"
    import torch
    import paper_2001_05585_b200 as T
    from paper_2001_05585_b200 import _capi
    lib = _capi.load()
    lib.tcr_enable_profiling_knobs()   # reads TCR_DEBUG_MODE=20 (knobs are never read implicitly)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    x = T.generate("uniform", 0, a.n, device=dev)
    res = torch.zeros(2, dtype=torch.float32, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    cfg = T.ReductionConfig(m=16, R=a.R, B=a.B, finalize=T.Finalize.tree).to_c()
    runs = []
    for rep in range(6):
        _capi.check(lib.tcr_single_pass_f16_async(C.c_void_p(x.data_ptr()), a.n, C.byref(cfg),
                                                  C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr()),
                                                  C.c_void_p(st.cuda_stream)))
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * (4 * 1024 + 4))()
        lib.tcr_debug_timestamps(buf, 4 * 1024 + 4)
        v = list(buf)
        ctas = [(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]) for i in range(1024) if v[4 * i] and v[4 * i + 1]]
        t0 = min(c[0] for c in ctas)
        starts = [c[0] - t0 for c in ctas]
        ends = [c[1] - t0 for c in ctas]
        last = [c for c in ctas if c[3] == 1][0]
        fin = (v[4 * 1024] - last[1]) / 1e3, (v[4 * 1024 + 1] - v[4 * 1024]) / 1e3
        runs.append({"ctas": len(ctas), "start_spread_us": (max(starts) - min(starts)) / 1e3,
                     "fin_ticket_us": fin[0], "fin_tree_us": fin[1],
                     "first_end_us": min(ends) / 1e3, "median_end_us": statistics.median(ends) / 1e3,
                     "last_end_us": max(ends) / 1e3, "tail_us": (max(ends) - statistics.median(ends)) / 1e3,
                     "finalise_us": (last[2] - last[1]) / 1e3, "span_us": (last[2] - t0) / 1e3})
        # clear for the next run
        lib.tcr_debug_timestamps  # noqa: B018
    for r in runs[1:]:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
