MRFG_ZOOM_PIT=1 timeout 600 python tools/zoom4_prior.py 2 1
MRFG_ZOOM_PIT=0 timeout 600 python tools/zoom4_prior.py 2 1
python - <<'PY'
import numpy as np
for m in (2, 1):
    a = np.load(f"gpurun_out/prior{m}_pit1.npy"); b = np.load(f"gpurun_out/prior{m}_pit0.npy")
    print(m, {k: int((a[k] == b[k]).sum()) for k in ("i1", "i2", "idf", "score", "pd", "evaluations")})
PY
timeout 900 python -m pytest tests/test_gpu_zoom.py tests/test_gpu_scale.py -q -x -k "slice or prior or config4 or exp3" 2>&1 | tail -2
