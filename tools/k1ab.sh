# K1 A/B on config 2 (bloch ms per step): E1/E2 tables vs MUFU, x-axis path
for cfg in "1 1" "1 0" "1 1" "1 0"; do set -- $cfg
MRFG_K1_XR=$1 MRFG_K1_TAB=$2 timeout 300 python bench.py --steps 2 --warmup 1 --no-zoom --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('xr=$1 tab=$2', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['breakdown_ms_per_step'].items()}, round(d['bloch_frac_of_fp32_peak_nominal'],4))"
done
