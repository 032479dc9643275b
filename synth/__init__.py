"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no GEMM, bias add, softmax,
k-best or compaction). It only draws numbers. Both sides of every parity
test read the tensors it returns, so oracle and kernels see identical inputs.

Generator: counter-based splitmix64. Element i of stream `stream` under seed
`seed` is

    key   = mix64(seed + stream * 0xD1B54A32D192ED03)      (host, Python int)
    z_i   = mix64(key + i * 0x9E3779B97F4A7C15)            (vectorised)

where mix64 is the splitmix64 finaliser. Because z_i depends only on the
global index i, a vocab shard regenerates its own slice of the one global W,
which makes shard-count invariance testable (SURVEY.md §8(d) "Generator").

Uniforms take the top 24 bits (exact in fp32). Normals use Box-Muller on pairs
of uniforms. bf16 values are produced by one fp32 -> bf16 round-to-nearest-even
(SURVEY.md §8(c) reading G9; the analogue of SPEC round_to_half).

Workload recipes (SURVEY.md §8(d) "Synthetic inputs", restated in DESIGN.md):
  zipf  : X ~ U(-1,1); W ~ N(0,1) * alpha / sqrt(H/3) with alpha=3 (logit std
          ~3); b_v = -0.5 ln(1+v) (Zipf unigram prior); prev_cost per sentence
          = B draws of -U(0,20) sorted descending; offsets[s] = s*B.
  flat  : alpha = 1 and b ~ N(0, 0.1^2)  (stress: near-ties, low peaks).
All tensors are generated with torch int64 arithmetic on any device; the
arithmetic wraps modulo 2^64 exactly like uint64 (checked against Python
big integers in tests/test_synth.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
STREAM_MUL = 0xD1B54A32D192ED03
BASE_SEED = 180509863

# streams
S_X, S_W, S_B, S_PREV, S_EOS, S_ALIVE, S_STATE = 1, 2, 3, 4, 5, 6, 7


def _s64(u: int) -> int:
    """uint64 -> int64 two's complement (torch has no full uint64 math)."""
    u &= MASK64
    return u - (1 << 64) if u >= (1 << 63) else u


def mix64_int(z: int) -> int:
    """splitmix64 finaliser on a Python int (reference for the tests)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    return mix64_int(seed + stream * STREAM_MUL)


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    """logical shift right on int64 holding uint64 bits."""
    return (z >> s) & ((1 << (64 - s)) - 1)


_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _mix64(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _srl(z, 30)) * _C1
    z = (z ^ _srl(z, 27)) * _C2
    return z ^ _srl(z, 31)


def raw64(seed: int, stream: int, start: int, count: int, device="cpu") -> torch.Tensor:
    """z_i for i in [start, start+count) as int64 holding uint64 bits."""
    key = stream_key(seed, stream)
    i = torch.arange(start, start + count, dtype=torch.int64, device=device)
    z = i * _s64(GOLDEN) + _s64(key)
    return _mix64(z)


def uniform24(seed, stream, start, count, device="cpu") -> torch.Tensor:
    """Integers j in [0, 2^24) (top 24 bits); u = j / 2^24 is exact in fp32."""
    return _srl(raw64(seed, stream, start, count, device), 40)


def uniform(seed, stream, start, count, lo=0.0, hi=1.0, device="cpu") -> torch.Tensor:
    j = uniform24(seed, stream, start, count, device).to(torch.float64)
    u = j * (1.0 / (1 << 24))
    return (lo + (hi - lo) * u).to(torch.float32)


def normal(seed, stream, start, count, device="cpu") -> torch.Tensor:
    """Box-Muller on the uniform pair (2p, 2p+1); element i uses pair i//2,
    cos branch for even i and sin branch for odd i."""
    p0 = start // 2
    p1 = (start + count + 1) // 2
    j = uniform24(seed, stream, 2 * p0, 2 * (p1 - p0), device).to(torch.float64)
    u1 = (j[0::2] + 1.0) * (1.0 / (1 << 24))  # (0, 1]
    u2 = j[1::2] * (1.0 / (1 << 24))
    r = torch.sqrt(-2.0 * torch.log(u1))
    t = 2.0 * math.pi * u2
    z = torch.stack([r * torch.cos(t), r * torch.sin(t)], dim=1).reshape(-1)
    off = start - 2 * p0
    return z[off:off + count].to(torch.float32)


def f32_to_bf16_rne(x: torch.Tensor) -> torch.Tensor:
    """fp32 -> bf16 bit pattern with round-to-nearest-even, returned as a
    torch.bfloat16 tensor (inputs are finite)."""
    b = x.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    rnd = ((b >> 16) & 1) + 0x7FFF
    h = ((b + rnd) >> 16) & 0xFFFF
    h = torch.where(h >= 0x8000, h - 0x10000, h).to(torch.int16)
    return h.view(torch.bfloat16)


@dataclass
class Workload:
    """One output-layer problem: S sentences x B beam rows, H hidden, V vocab."""
    name: str
    H: int
    V: int
    S: int
    B: int
    k: int
    dtype: str = "bf16"          # "bf16" or "f32"
    dist: str = "zipf"           # "zipf" or "flat"
    seed: int = BASE_SEED
    extra: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return self.S * self.B


# BASELINE.json configs. cfg4's H is assumed 1024.
CONFIGS = {
    "tiny": Workload("tiny", H=64, V=1000, S=4, B=2, k=2, dtype="f32", seed=BASE_SEED + 1),
    "greedy": Workload("greedy", H=512, V=60000, S=128, B=1, k=1, seed=BASE_SEED + 2),
    "beam": Workload("beam", H=1024, V=90000, S=128, B=5, k=5, seed=BASE_SEED + 3),
    "trace": Workload("trace", H=1024, V=90000, S=1280, B=5, k=5, seed=BASE_SEED + 4),
    "shard": Workload("shard", H=1024, V=256000, S=1024, B=12, k=12, seed=BASE_SEED + 5),
}


def gen_X(w: Workload, row0: int = 0, rows: int | None = None, device="cpu"):
    rows = w.N - row0 if rows is None else rows
    x = uniform(w.seed, S_X, row0 * w.H, rows * w.H, -1.0, 1.0, device).view(rows, w.H)
    return f32_to_bf16_rne(x) if w.dtype == "bf16" else x


def gen_W(w: Workload, v0: int = 0, vcount: int | None = None, device="cpu"):
    """Rows [v0, v0+vcount) of the global W [V, H]."""
    vcount = w.V - v0 if vcount is None else vcount
    alpha = 3.0 if w.dist == "zipf" else 1.0
    scale = alpha / math.sqrt(w.H / 3.0)
    z = normal(w.seed, S_W, v0 * w.H, vcount * w.H, device).view(vcount, w.H)
    z = (z.to(torch.float64) * scale).to(torch.float32)
    return f32_to_bf16_rne(z) if w.dtype == "bf16" else z


def gen_b(w: Workload, v0: int = 0, vcount: int | None = None, device="cpu"):
    vcount = w.V - v0 if vcount is None else vcount
    if w.dist == "zipf":
        v = torch.arange(v0, v0 + vcount, dtype=torch.float64, device=device)
        return (-0.5 * torch.log1p(v)).to(torch.float32)
    return (normal(w.seed, S_B, v0, vcount, device).to(torch.float64) * 0.1).to(torch.float32)


def gen_prev_cost(w: Workload, device="cpu"):
    u = uniform(w.seed, S_PREV, 0, w.N, 0.0, 20.0, device).view(w.S, w.B)
    pc = -u
    pc, _ = torch.sort(pc, dim=1, descending=True)
    return pc.reshape(-1).contiguous()


def gen_offsets(w: Workload, device="cpu"):
    return (torch.arange(w.S + 1, dtype=torch.int32, device=device) * w.B).contiguous()


def gen_alive(seed: int, N: int, p: float, device="cpu") -> torch.Tensor:
    """i.i.d. survival mask with probability p (u8 0/1)."""
    j = uniform24(seed, S_ALIVE, 0, N, device)
    return (j < int(p * (1 << 24))).to(torch.uint8)


def gen_bytes(seed: int, stream: int, nbytes: int, device="cpu") -> torch.Tensor:
    """nbytes of pseudo-random bytes (state columns for compaction tests)."""
    n8 = (nbytes + 7) // 8
    z = raw64(seed, stream, 0, n8, device)
    return z.view(torch.uint8)[:nbytes].clone()


def eos_schedule(seed: int, S: int, B: int, p: float = 1.0 / 20.0, cap: int = 60):
    """cfg4 schedule (SURVEY.md §8(d) "Config 4 schedule"): sentence length
    L_s ~ Geometric(p) on {1,2,...} capped at `cap`; hypothesis j of sentence
    s finishes at f_{s,j} = L_s + j. Returns int64 tensor f[S, B]."""
    u = uniform(seed, S_EOS, 0, S, device="cpu").to(torch.float64)
    u = torch.clamp(u, min=1.0 / (1 << 25))
    L = torch.floor(torch.log(u) / math.log1p(-p)).to(torch.int64) + 1
    L = torch.clamp(L, 1, cap)
    return L[:, None] + torch.arange(B, dtype=torch.int64)[None, :]
