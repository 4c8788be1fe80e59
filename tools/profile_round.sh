#!/bin/bash
# Round profile set (run on the GPU box from the repo root; outputs in gpurun_out/).
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python tools/bench_config5_zoom.py > $O/config5_zoom.json 2> $O/config5_zoom.err; echo "c5zoom rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-zoom --atoms 4194304"
timeout 600 $B > $O/short.json 2>&1; echo "short rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-zoom > /dev/null 2>&1; echo "launches rc=$?"
# gpurun copies back <= 64 MiB: export the pages as CSV on the box and keep
# only small reports
export_rep() {
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_sass.csv 2>/dev/null
  gzip -f $O/$1_sass.csv $O/$1_raw.csv
  [ $(stat -c %s $O/$1.ncu-rep) -gt 12000000 ] && rm -f $O/$1.ncu-rep
}
for spec in "k2:regex:k_match_sm100_2cta:4" "k1:regex:k_bloch_rows2:4" "k3:regex:^k_rescreen32\$:0"; do
  IFS=: read name kind pat skip <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$pat" -s $skip -c 1 \
      -o $O/ncu_$name $B > $O/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  export_rep ncu_$name
done
timeout 600 python tools/zoom4_quick.py 4096 1e-5 > $O/zoom4.json 2>&1; echo "zoom4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zoom -s 1 -c 1 \
    -o $O/ncu_k5 python tools/zoom4_once.py > $O/ncu_k5.log 2>&1; echo "ncu k5 rc=$?"
export_rep ncu_k5
du -sh $O
