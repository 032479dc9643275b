"""Probe the MXFP4 fused kernel at one vocabulary size (run one size per
process: an illegal instruction poisons the CUDA context). With N = 128 rows
(one M-tile, 148 vocab splits), V = 148 x w gives every CTA one tile of
width w. Integer-regime inputs: the logits must equal the oracle's exactly.

  python tools/f4_probe.py V     (one JSON line)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402


def main():
    V = int(sys.argv[1])
    N, H = int(os.environ.get("PROBE_N", "128")), 256
    rng = np.random.default_rng(1)
    X = rng.integers(-8, 9, (N, H)).astype(np.float32)
    X[:, 0] = 448.0
    X8, xs = O.quantize_rows_e4m3(X)
    grid = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    Wv = rng.choice(grid, (V, H)) * rng.choice([-1.0, 1.0], (V, H))
    Wv = Wv * np.repeat(2.0 ** rng.integers(-2, 3, (V, H // 32)), 32, axis=1)
    b = rng.integers(-4, 5, V).astype(np.float32)
    dev = torch.device("cuda", 0)
    W4, sf = amun.quantize_mxfp4(torch.from_numpy(Wv.astype(np.float32)).to(dev))
    ol = amun.OutputLayer(H, V, dtype="mxfp4", k_max=4, max_rows=N, max_sentences=N)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    out = {"V": V, "N": N}
    try:
        L = ol.debug_logits_mxfp4(t(X8), t(xs), W4, sf, t(b))
        torch.cuda.synchronize()
        want = O.add_bias(O.gemm(O.dequant_rows_e4m3(X8, xs), Wv), O.as_f64(b))
        got = L.cpu().numpy().astype(np.float64)
        bad = np.argwhere(got != want)
        out.update(ok=True, exact=bool(len(bad) == 0), n_bad=int(len(bad)),
                   bad_cols=sorted(set(int(c) for c in bad[:2000, 1]))[:40])
    except Exception as e:  # noqa: BLE001
        out.update(ok=False, error=str(e).splitlines()[0][:120])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
