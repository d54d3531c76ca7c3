"""CPU-oracle timing beside the GPU numbers (SURVEY §8(d) "Oracle timing beside
it"): configs c1, c2, c3 in fixed and double mode, all host cores and one
thread; c4 / c5 extrapolated from c3 (labelled).  Test infrastructure only
(it runs oracle/); prints one JSON object.  Usage: python tools/oracle_timing.py"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_2212_00488_b200 import synth  # noqa: E402


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def time_one(L, R, D, K, mode, nthreads, budget=6.0, max_runs=20):
    p = oracle.params(k_scale=K)
    n, t0 = 0, time.perf_counter()
    while True:
        oracle.pipeline(L, R, D, p, mode, nthreads=nthreads, stages=("out",))
        n += 1
        el = time.perf_counter() - t0
        if el >= budget or n >= max_runs:
            return el / n


def main():
    nc = cores()
    cfgs = {"c1": (64, 48, 16, 1, lambda: synth.shift_pair(64, 48, 5, seed=0)),
            "c2": (450, 375, 64, 1, lambda: synth.scene(450, 375, 64, seed=1)[:2]),
            "c3": (1436, 992, 145, 2, lambda: synth.scene(1436, 992, 145, seed=0)[:2])}
    res = {"cpu": cpu_model(), "cores": nc, "configs": {}}
    for name, (W, H, D, K, gen) in cfgs.items():
        L, R = gen()
        row = {}
        for mode in ("fixed", "double"):
            for nt in (nc, 1):
                if name == "c3" and nt == 1 and mode == "double":
                    continue  # > a minute; the fixed 1-thread figure stands for it
                s = time_one(L, R, D, K, mode, nt, budget=2.0 if nt == 1 else 6.0,
                             max_runs=1 if (name == "c3" and nt == 1) else 20)
                row[f"{mode}_threads{nt}_s_per_frame"] = s
        res["configs"][name] = row
    c3 = res["configs"]["c3"]["fixed_threads%d_s_per_frame" % nc]
    res["extrapolated"] = {"c4_256_frames_s": 256 * c3, "c5_one_frame_s": 8 * c3,
                           "note": "c4 = 256 x c3; c5 = 8 x c3 (4x pixels, 2x disparities); "
                                   "fixed mode, all cores; not measured"}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
