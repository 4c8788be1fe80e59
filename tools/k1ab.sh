# K1 A/B on config 2 (Bloch ms per step).  Arguments: configs
# K1:APT:MINB:HB:ST -- producer (pairs = atom-pair kernel, rows2 = packed
# (x, y) kernel), atoms per thread, resident blocks per SM, echo steps
# buffered per store, staged stores.  Default: a small set.
[ $# -eq 0 ] && set -- pairs:4:2:8:1 pairs:8:2:8:1 pairs:4:3:8:1 pairs:4:2:8:0 rows2:4:2:8:1 pairs:4:2:8:1
for cfg in "$@"; do IFS=: read k1 apt minb hb st <<< "$cfg"
MRFG_K1=$k1 MRFG_K1_APT=$apt MRFG_K1_MINB=$minb MRFG_K1_HB=$hb MRFG_K1_ST=$st timeout 300 python bench.py --steps 2 --warmup 1 --no-zoom --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['breakdown_ms_per_step'].items()}, round(d['bloch_frac_of_fp32_peak_nominal'],4))"
done
