"""Synthetic sources for benches and tests.

Zipf over 256 symbols, p_k proportional to (k+1)^-s, sampled by inverse CDF
over a counter-based hash: byte i = #{k < 255 : cdf[k] <= u_i},
u_i = splitmix64(seed ^ i) >> 32. The device generator
(csrc/synth.cu, ilans_synth_bytes_dev) and ``synth_host`` below produce
identical bytes, so any shard can be regenerated anywhere.
"""

from __future__ import annotations

import numpy as np

# exponents solved for target entropies
ZIPF_S_FOR_ENTROPY = {1.0: 2.971782, 2.0: 2.151942, 4.0: 1.479920, 6.0: 1.049543,
                      7.9: 0.323186}
DEFAULT_S = 1.1  # config 2/3 default, H ~= 5.77 bits/byte


def zipf_probs(s: float, n: int = 256) -> np.ndarray:
    p = (np.arange(n) + 1.0) ** -s
    return p / p.sum()


def zipf_cdf_u32(s: float) -> np.ndarray:
    """u32 thresholds: cdf[k] = floor(2^32 * P(X <= k)), k < 255; cdf[255] = max."""
    c = np.cumsum(zipf_probs(s))
    cdf = np.minimum(np.floor(c * 2.0**32), 2.0**32 - 1).astype(np.uint64)
    cdf[255] = 2**32 - 1
    return cdf.astype(np.uint32)


def entropy_bits(p: np.ndarray) -> float:
    p = p[p > 0]
    return float(-(p * np.log2(p)).sum())


_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = z + _M1
    z = (z ^ (z >> np.uint64(30))) * _M2
    z = (z ^ (z >> np.uint64(27))) * _M3
    return z ^ (z >> np.uint64(31))


def synth_host(n: int, s: float = DEFAULT_S, seed: int = 1234, first: int = 0) -> np.ndarray:
    """Host twin of ilans_synth_bytes_dev (numpy, ~100 MB/s)."""
    cdf = zipf_cdf_u32(s)[:255]
    out = np.empty(n, dtype=np.uint8)
    step = 1 << 22
    with np.errstate(over="ignore"):
        for a in range(0, n, step):
            b = min(n, a + step)
            i = np.arange(first + a, first + b, dtype=np.uint64)
            u = (splitmix64(np.uint64(seed) ^ i) >> np.uint64(32)).astype(np.uint32)
            out[a:b] = np.searchsorted(cdf, u, side="right").astype(np.uint8)
    return out


def synth_device(n: int, s: float = DEFAULT_S, seed: int = 1234, first: int = 0, out=None,
                 device=None):
    """Generate n bytes on the GPU (torch uint8 tensor, 16-byte aligned)."""
    import torch

    from . import _lib

    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if out is None:
        out = torch.empty(max(16, n), dtype=torch.uint8, device=dev)
    cdf = torch.from_numpy(zipf_cdf_u32(s).view(np.int32).copy()).to(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check_dev(_lib.lib.ilans_synth_bytes_dev(out.data_ptr(), int(n), int(seed), int(first),
                                                  cdf.data_ptr(), stream), "synth")
    torch.cuda.current_stream(dev).synchronize()  # cdf must outlive the launch
    return out
