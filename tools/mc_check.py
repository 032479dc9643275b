"""Parity of the W-multicast cluster experiment (AMUN_MC=4): a batch of exactly
4 M-tiles (N = 512) through amun_output_layer against the oracle, and
bit-identity with the unicast kernel.  python tools/mc_check.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import synth  # noqa: E402
from tests.compare import compare_kbest  # noqa: E402

os.environ["AMUN_MC"] = "4"
import paper_1805_09863_b200 as amun  # noqa: E402

dev = torch.device("cuda", 0)
w = synth.Workload("mc", H=1024, V=20011, S=128, B=4, k=5, seed=synth.BASE_SEED + 555)
X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
ol = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
i1, c1 = ol(X, W, b, pc, off, w.k)
torch.cuda.synchronize()
os.environ["AMUN_MC"] = "0"
ol0 = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
i0, c0 = ol0(X, W, b, pc, off, w.k)
torch.cuda.synchronize()
L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w))), O.as_f64(synth.gen_b(w)))
logp = O.log_softmax(L)
pcd = O.as_f64(synth.gen_prev_cost(w))
_, _, oc64, nxt = O.kbest_sentences(logp, pcd, off.cpu().numpy(), w.k)
rep = compare_kbest(i1.cpu().numpy(), c1.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v], oc64,
                    np.full(w.S, w.k), "bf16", w.V, o_next=nxt)
print("mc=4 parity:", rep, "identical to unicast:", bool(torch.equal(i1, i0) and torch.equal(c1, c0)))
