"""Seeded request traces shaped like the paper's workloads.

* Lengths: PAPER.md Table 4 gives means/medians; the lognormal fit
  mu = ln(median), sigma = sqrt(2 ln(mean/median)) is used for
  ShareGPT/Alpaca-like traces, truncated to [1, 4096] ("truncating inputs
  to a maximum length of 4096"). LongBench cannot be fit that way (mean <
  median, SURVEY reading A26), so long prompts are uniform U{6144..8192}.
* Arrivals: Poisson at a fixed rate -> i.i.d. exponential inter-arrival
  gaps, floored to integer nanoseconds.
* Prompt tokens: i.i.d. uniform over the vocabulary (random-init weights, no
  tokenizer).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np


@dataclass
class Request:
    req_id: int
    arrival_ns: int
    prompt_len: int          # S
    output_len: int          # G, includes the prefill token (reading A7)
    prompt: Optional[np.ndarray] = None  # int32 [S]


@dataclass(frozen=True)
class LengthDist:
    kind: str                # "uniform" | "lognormal"
    a: float                 # uniform lo | lognormal median
    b: float                 # uniform hi | lognormal mean
    lo: int = 1
    hi: int = 4096

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        if self.kind == "uniform":
            return rng.integers(int(self.a), int(self.b) + 1, size=n).astype(np.int64)
        mu = np.log(self.a)
        sigma = np.sqrt(2.0 * np.log(self.b / self.a))
        out = np.empty(n, dtype=np.int64)
        filled = 0
        while filled < n:
            x = np.floor(rng.lognormal(mu, sigma, size=2 * (n - filled) + 8)).astype(np.int64)
            x = x[(x >= self.lo) & (x <= self.hi)]
            take = min(len(x), n - filled)
            out[filled:filled + take] = x[:take]
            filled += take
        return out


# Table 4: (In_avg, In_med, Out_avg, Out_med, SLO_TTFT s, SLO_TPOT s)
TABLE4 = {
    "alpaca": (20.63, 17.00, 163.80, 119.00, 1.0, 0.100),
    "sharegpt": (343.76, 148.00, 237.20, 152.0, 5.0, 0.100),
    "longbench": (2686.89, 2736.50, 101.78, 19.0, 15.0, 0.100),
}

PRESETS = {
    # BASELINE.json configs[1]: prompts 512-2k, outputs 128-512
    "8b-cycle": (LengthDist("uniform", 512, 2048), LengthDist("uniform", 128, 512)),
    # configs[2]/[3]: chat-like (ShareGPT fit)
    "sharegpt": (LengthDist("lognormal", 148.0, 343.76), LengthDist("lognormal", 152.0, 237.20)),
    "alpaca": (LengthDist("lognormal", 17.0, 20.63), LengthDist("lognormal", 119.0, 163.80)),
    # configs[4]: long prompts (A26) and LongBench-like outputs
    "long": (LengthDist("uniform", 6144, 8192, 1, 8192), LengthDist("lognormal", 19.0, 101.78, 1, 1024)),
    # configs[0]: tiny decoder, prompts 32-128, 16 output tokens
    "tiny": (LengthDist("uniform", 32, 128), LengthDist("uniform", 16, 16)),
}


def poisson_arrivals_ns(rng: np.random.Generator, n: int, rate_per_s: float, t0_ns: int = 0) -> np.ndarray:
    gaps = np.floor(rng.exponential(1e9 / rate_per_s, size=n)).astype(np.int64)
    return t0_ns + np.cumsum(gaps)


def make_trace(preset: str, n: int, seed: int, rate_per_s: Optional[float] = None,
               vocab: Optional[int] = None) -> List[Request]:
    """n requests; arrivals at time 0 if rate is None, else Poisson(rate)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 7])))
    din, dout = PRESETS[preset]
    s = din.sample(rng, n)
    g = dout.sample(rng, n)
    if rate_per_s is None:
        arr = np.zeros(n, dtype=np.int64)
    else:
        arr = poisson_arrivals_ns(rng, n, rate_per_s)
    reqs = []
    for i in range(n):
        prompt = None
        if vocab is not None:
            prompt = rng.integers(0, vocab, size=int(s[i])).astype(np.int32)
        reqs.append(Request(i, int(arr[i]), int(s[i]), int(g[i]), prompt))
    return reqs


def random_prompts(seed: int, lengths, vocab: int) -> List[np.ndarray]:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 11])))
    return [rng.integers(0, vocab, size=int(n)).astype(np.int32) for n in lengths]
