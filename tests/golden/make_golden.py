"""Regenerate tests/golden/* from the reference's recorded runs (run where
/root/reference exists; the fixtures are committed and nothing at test time
reads /root/reference).

  exp2.json       runs/exp2/{targets,zoom,brute}.csv   (25 targets, N=500 seed 1)
  exp1_ccdf.npz   runs/exp1/cc_vs_df.csv               (first 1,200 rows: 2 T1/T2 pairs x 600 df)
  exp3_slice.npz  data/slice64.csv + runs/exp3/results_noprior.csv + t1/t2/df_map_noprior.csv
"""
import csv
import json
import os

import numpy as np

REF = "/root/reference/proj"
OUT = os.path.dirname(os.path.abspath(__file__))


def rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def main():
    R = REF + "/runs/exp2/"
    t = [[float(r["t1_ms"]), float(r["t2_ms"]), float(r["df_hz"])] for r in rows(R + "targets.csv")]
    z = [[float(r["t1_ms"]), float(r["t2_ms"]), float(r["df_hz"]), float(r["pd"]), float(r["score"]),
          int(r["evals"])] for r in rows(R + "zoom.csv")]
    b = [[float(r["t1_ms"]), float(r["t2_ms"]), float(r["df_hz"]), float(r["pd"]), float(r["score"]),
          int(r["evals"])] for r in rows(R + "brute.csv")]
    with open(os.path.join(OUT, "exp2.json"), "w") as f:
        json.dump({"source": "proj/runs/exp2/{targets,zoom,brute}.csv (schedule n=500 seed=1; grid "
                             "500:2000:10 x 200:800:10 x -30:450:2; df_coarse=2)",
                   "targets": t, "zoom": z, "brute": b}, f, indent=0)

    cc = rows(REF + "/runs/exp1/cc_vs_df.csv")[:1200]
    np.savez_compressed(os.path.join(OUT, "exp1_ccdf.npz"),
                        t1_ms=np.array([float(r["t1_ms"]) for r in cc]),
                        t2_ms=np.array([float(r["t2_ms"]) for r in cc]),
                        df_hz=np.array([float(r["df_hz"]) for r in cc]),
                        cc_text=np.array([r["cc"] for r in cc]))

    sl = rows(REF + "/data/slice64.csv")
    res = {int(r["id"]): r for r in rows(REF + "/runs/exp3/results_noprior.csv")}
    resp = {int(r["id"]): r for r in rows(REF + "/runs/exp3/results_prior.csv")}
    n = len(sl)
    maps = {k: np.loadtxt(REF + f"/runs/exp3/{k}_map_noprior.csv", delimiter=",").reshape(-1)
            for k in ("t1", "t2", "df")}
    np.savez_compressed(
        os.path.join(OUT, "exp3_slice.npz"),
        mask=np.array([int(r["mask"]) for r in sl], dtype=np.uint8),
        t1_ms=np.array([float(r["t1_ms"]) for r in sl]), t2_ms=np.array([float(r["t2_ms"]) for r in sl]),
        df_hz=np.array([float(r["df_hz"]) for r in sl]), pd=np.array([float(r["pd"]) for r in sl]),
        evals_noprior=np.array([int(res[i]["evals"]) if i in res else 0 for i in range(n)]),
        evals_prior=np.array([int(resp[i]["evals"]) if i in resp else 0 for i in range(n)]),
        t1_map=maps["t1"], t2_map=maps["t2"], df_map=maps["df"])


if __name__ == "__main__":
    main()
