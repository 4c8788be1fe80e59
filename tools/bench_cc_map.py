"""§8(f) row 1: cc_map over the config-2 lattice (BASELINE configs[1]: T1
100-5000/10, T2 20-2000/5, df -250..250/1 = 97,658,427 atoms, N = 1000).

Times (CUDA events around the ABI call, host output included) the fused FP32
kernel (precision 32: K1 row kernel with the query dot fused, 4 B/atom out)
over the whole lattice and the bit-exact FP64 pipeline (precision 64) over a
sample, checks the FP32 map against FP64 on that sample, and writes the .mrfc
file of the whole lattice (timed separately: disk-bound).  One JSON line.
Usage: python tools/bench_cc_map.py [sample_atoms]
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05393_b200 as P  # noqa: E402


def main():
    sample = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    n = 1000
    s = P.baseline_schedule(n, 1)
    g = P.grid_inclusive((100.0, 5000.0, 10.0), (20.0, 2000.0, 5.0), (-250.0, 250.0, 1.0))
    total = P.grid_total(g)
    with P.Context(s) as c:
        # a noisy config-2 tissue fingerprint as the query
        fp = c.simulate(np.array([[1.23, 0.087, 17.0]]), precision=64)[0]
        fp = P.add_noise(fp, float(np.linalg.norm(fp) / np.sqrt(n) / 30.0), 4242)
        c.cc_map(fp, g, 0, 1 << 20, precision=32)  # warm-up (tables)
        t0 = time.perf_counter()
        fast = c.cc_map(fp, g, precision=32)
        t_fast = time.perf_counter() - t0
        first = total // 2 - sample // 2
        c.cc_map(fp, g, first, 1024, precision=64)
        t0 = time.perf_counter()
        exact = c.cc_map(fp, g, first, sample, precision=64)
        t_exact = time.perf_counter() - t0
        err = float(np.abs(fast[first:first + sample].astype(np.float64) - exact).max())
        with tempfile.TemporaryDirectory() as d:
            t0 = time.perf_counter()
            c.cc_map_to_file(fp, g, os.path.join(d, "cfg2.mrfc"), precision=32)
            t_file = time.perf_counter() - t0
            size = os.path.getsize(os.path.join(d, "cfg2.mrfc"))
    # algorithmic work: 37 flop/atom-step Bloch + 8 flop/atom-step complex dot
    flop = total * n * (37 + 8)
    print(json.dumps({
        "metric": "cc_map atoms/s (config-2 lattice, N=1000)", "atoms": total,
        "fp32_s": t_fast, "fp32_atoms_per_s": total / t_fast,
        "fp32_tflops_algorithmic": flop / t_fast / 1e12,
        "fp64_sample_atoms": sample, "fp64_atoms_per_s": sample / t_exact,
        "fp32_vs_fp64_max_abs_err": err, "argmax_flat": int(np.argmax(fast)),
        "mrfc_file_s": t_file, "mrfc_bytes": size,
    }))


if __name__ == "__main__":
    main()
