#!/bin/bash
# Round profile set (run on the GPU box from the repo root; outputs in gpurun_out/).
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python tools/bench_config5_zoom.py > $O/config5_zoom.json 2> $O/config5_zoom.err; echo "c5zoom rc=$?"
# the short run: one timed full-lattice scan (subspace screening needs whole lattice rows)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-zoom --no-full"
timeout 600 $B > $O/short.json 2> $O/short.err; echo "short rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv \
    $B > /dev/null 2>&1; echo "launches rc=$?"
# one ncu --set full capture per kernel (details, raw, SASS source and
# per-instruction stall pages; tools/ncu_one.sh writes gpurun_out/ncu/)
CMD="$B" bash tools/ncu_one.sh k_match_sm100_2cta 4 ncu_k2
CMD="$B" bash tools/ncu_one.sh k_bloch_pairs_st 4 ncu_k1
CMD="$B" bash tools/ncu_one.sh "^k_rescreen32\$" 0 ncu_k3
CMD="$B" bash tools/ncu_one.sh k_project 600 ncu_proj
# K2 in the full-length regime (MRFG_SUBSPACE=0)
MRFG_SUBSPACE=0 CMD="$B" bash tools/ncu_one.sh k_match_sm100_2cta 4 ncu_k2_full
timeout 600 python tools/zoom4_quick.py 4096 1e-5 > $O/zoom4.json 2>&1; echo "zoom4 rc=$?"
CMD="python tools/zoom4_once.py" bash tools/ncu_one.sh k_zoom 1 ncu_k5
MRFG_ZOOM_STATS=1 ZOOM_REPS=1 timeout 600 python tools/zoom4_quick.py 4096 1e-5 2>&1 | grep "mrfg zoom" | tail -1 > $O/zoom4_stats.txt
python tools/k2_traffic.py gpurun_out/ncu/ncu_k2_raw.csv.gz $O/short.json > $O/k2_traffic.json; echo "traffic rc=$?"
du -sh $O gpurun_out/ncu
