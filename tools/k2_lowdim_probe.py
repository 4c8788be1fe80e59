"""What would the matching stage cost in a 2r-dimensional subspace?
Times K2 (+ the stored-dictionary operand kernel and K3) through the public
stored-dictionary scan with n = r "timepoints" (2r real dimensions, padded to
one 64-wide K block): 4,096 unit queries against `atoms` random unit entries,
the queries being noisy copies of entries.  Extrapolates the K2 time to the
config-2 lattice (97,658,427 atoms).  DESIGN.md 7 (per-off-resonance subspace
screening) cites the result.
Usage: python tools/k2_lowdim_probe.py [r] [atoms]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05393_b200 as P  # noqa: E402


def main():
    import torch
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    atoms = int(sys.argv[2]) if len(sys.argv) > 2 else 8_000_000
    nq = 4096
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    d = torch.randn(atoms, r, 2, device=dev, generator=g, dtype=torch.float32)
    d /= d.flatten(1).norm(dim=1).view(-1, 1, 1)
    pick = torch.randint(0, atoms, (nq,), device=dev, generator=g)
    q = d[pick].double() + 0.03 * torch.randn(nq, r, 2, device=dev, generator=g, dtype=torch.float64)
    out = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
    # a schedule of r steps only provides the context (n = r)
    s = P.dgs.baseline_schedule(r, 1)
    stream = torch.cuda.current_stream(dev)
    res = {}
    with P.Context(s) as c:
        c.set_stream(stream.cuda_stream)
        for _ in range(2):
            st = c.scan_dict_device(d.data_ptr(), atoms, q.data_ptr(), nq, out.data_ptr())
        torch.cuda.synchronize()
        res = {"r": r, "atoms": atoms, "voxels": nq, "gemm_ms": st.gemm_ms, "bloch_or_operand_ms": st.bloch_ms,
               "rerank_ms": st.rerank_ms, "total_ms": st.total_ms, "candidates": st.candidates,
               "k2_ms_extrapolated_to_97.66M_atoms": st.gemm_ms * 97_658_427 / atoms}
        m = np.frombuffer(out.cpu().numpy().tobytes(), dtype=np.dtype([("flat", np.int64), ("score", np.float64)]))
        res["recovered"] = int((m["flat"] == pick.cpu().numpy()).sum())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
