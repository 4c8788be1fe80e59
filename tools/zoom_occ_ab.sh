# K5 block shape / register budget and table layout on config 4 (ms, voxels/s, identity with all-FP64)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
for cfg in "256 1 1" "256 1 0" "128 3 1" "128 3 0" "256 1 1"; do set -- $cfg
  MRFG_ZOOM_SY=$3 MRFG_ZOOM_BS=$1 MRFG_ZOOM_MINB=$2 timeout 300 python tools/zoom4_quick.py 4096 1e-5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bs=$1 minb=$2 sy=$3', round(d['1e-5']['ms'],2), int(d['1e-5']['voxels_per_s']), d['1e-5']['ms_all'])"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
