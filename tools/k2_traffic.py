"""DRAM traffic of one K2 launch from an ncu --set full capture (the raw page
exported by tools/ncu_one.sh) -> the JSON bench.py reads
(profiles/r02_k2_traffic.json).  The capture comes from the short bench run
(`--atoms 4194304`), whose launches have the same shape as the full run's.
Usage: python tools/k2_traffic.py ncu_k2_raw.csv.gz short_bench.json
"""
import csv
import gzip
import json
import sys


def main():
    raw, short = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(gzip.open(raw, "rt")))
    names, vals = rows[0], rows[2]
    m = dict(zip(names, vals))
    units = dict(zip(names, rows[1]))
    scale = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}
    rd = float(m["dram__bytes_read.sum"]) * scale[units["dram__bytes_read.sum"].lower()]
    wr = float(m["dram__bytes_write.sum"]) * scale[units["dram__bytes_write.sum"].lower()]
    with open(short) as f:
        line = [ln for ln in f.read().splitlines() if ln.startswith("{")][-1]
    b = json.loads(line)
    atoms = b["roofline"]["atoms_per_launch"]
    nq, n = b["config"]["voxels"], b["config"]["timepoints"]
    kpad = (b["roofline"].get("k_dims", 2 * n) + 63) // 64 * 64  # operand width K2 sees
    arows = (atoms + 255) // 256 * 256
    qrows = (2 * nq + 255) // 256 * 256
    alg = (arows + qrows) * kpad * 2
    out = {"kernel": "k_match_sm100_2cta (K2)",
           "source": "ncu --set full --clock-control none, one k_match_sm100_2cta launch of python bench.py "
                     "--steps 1 --warmup 1 --no-cpu-baseline --no-zoom --no-full (-s 4 -c 1), "
                     "profiles/r02_ncu/ncu_k2_raw.csv.gz",
           "chunk_atoms": atoms, "voxels": nq, "timepoints": n,
           "dram_bytes_read": rd, "dram_bytes_write": wr,
           "dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": alg,
           "note": f"fp16 atom operand ({arows} x {kpad} x 2 B) + query operand ({qrows} x {kpad} x 2 B); "
                   f"traffic/algorithmic = {(rd + wr) / alg:.3f}", "round": 2}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
