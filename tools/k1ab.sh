# K1 A/B on config 2 (Bloch ms per step): x-axis RF path on/off, resident blocks per SM
for cfg in "1 2" "0 2" "1 3" "1 2"; do set -- $cfg
MRFG_K1_XR=$1 MRFG_K1_MINB=$2 timeout 300 python bench.py --steps 2 --warmup 1 --no-zoom --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('xr=$1 minb=$2', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['breakdown_ms_per_step'].items()}, round(d['bloch_frac_of_fp32_peak_nominal'],4))"
done
