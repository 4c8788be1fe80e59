#!/bin/bash
# One ncu --set full capture of kernel regex $1 (skip $2 launches) over a
# short config-2 bench; exports details/raw/source pages into gpurun_out/$3_*.
set -u
O=gpurun_out/ncu; mkdir -p $O
PAT=$1; SKIP=${2:-2}; NAME=${3:-k}; shift 3 || true
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-zoom --atoms 4194304"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$PAT" -s $SKIP -c 1 \
    -o $O/$NAME ${CMD:-$B} > $O/$NAME.log 2>&1; echo "ncu $NAME rc=$?"
ncu -i $O/$NAME.ncu-rep --page details --csv > $O/${NAME}_details.csv 2>/dev/null
ncu -i $O/$NAME.ncu-rep --page raw --csv > $O/${NAME}_raw.csv 2>/dev/null
ncu -i $O/$NAME.ncu-rep --page source --csv --print-source sass > $O/${NAME}_sass.csv 2>/dev/null
# per-instruction stall reasons (+ executed counts come from the _sass page, same row order)
ST=smsp__pcsamp_warps_issue_stalled
ncu -i $O/$NAME.ncu-rep --page source --csv --print-source sass --metrics ${ST}_long_scoreboard,${ST}_wait,${ST}_math_pipe_throttle,${ST}_short_scoreboard,${ST}_not_selected,${ST}_selected,${ST}_no_instructions,${ST}_branch_resolving,${ST}_dispatch_stall,${ST}_mio_throttle,${ST}_lg_throttle,${ST}_barrier,${ST}_membar,${ST}_drain,${ST}_imc_miss,${ST}_tex_throttle,${ST}_sleeping,${ST}_misc > $O/${NAME}_stalls.csv 2>/dev/null
gzip -f $O/${NAME}_stalls.csv
gzip -f $O/${NAME}_sass.csv $O/${NAME}_raw.csv
[ $(stat -c %s $O/$NAME.ncu-rep) -gt 12000000 ] && rm -f $O/$NAME.ncu-rep
ls -la $O
