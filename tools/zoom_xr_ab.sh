timeout 900 python -m pytest tests/test_gpu_zoom.py -q -x 2>&1 | tail -2
for xr in 1 0 1; do MRFG_ZOOM_XR=$xr timeout 300 python tools/zoom4_quick.py 4096 1e-5 -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('xr=$xr', d['1e-5']['ms'], d['1e-5']['voxels_per_s'], d['1e-5'].get('identical_to_-1'))"; done
