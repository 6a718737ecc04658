"""Counter-based synthetic inputs for BASELINE config 5.

Config 5 is n = 2^31 int64 keys uniform over the full int64 range with 10%
of positions overwritten by one repeated value, sharded evenly over the
GPUs.  A counter-based generator (splitmix64 of the global index) lets every
rank build its own shard on its device and lets any checker regenerate any
key.  Choices the BASELINE text leaves open, recorded here and in DESIGN.md:
  * key_i = splitmix64(SEED_MIX + i), SEED_MIX = 4 << 56 (seed 4);
  * position i is overwritten iff the 53-bit uniform from
    splitmix64(SALT + i) is < 0.1 (Bernoulli(0.1), not exactly floor(0.1 n));
  * the repeated value is splitmix64(4).
Float-free integer arithmetic, identical on host (oracle.splitmix64) and
device.
"""

from __future__ import annotations

import torch

SEED_MIX = 4 << 56
SALT = 0x5A5A5A5A << 32
_TENTH_53 = int(0.1 * (1 << 53))


def _i64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= 1 << 63 else x


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic)."""
    z = x + _i64(0x9E3779B97F4A7C15)
    z = (z ^ _lsr(z, 30)) * _i64(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * _i64(0x94D049BB133111EB)
    return z ^ _lsr(z, 31)


def repeated_value() -> int:
    return int(splitmix64(torch.tensor([4], dtype=torch.int64))[0])


def config5_keys(offset: int, count: int, n_total: int, device="cuda", chunk: int = 1 << 27) -> torch.Tensor:
    """Keys for global positions [offset, offset + count) of config 5."""
    assert 0 <= offset and offset + count <= n_total
    out = torch.empty(count, dtype=torch.int64, device=device)
    rep = repeated_value()
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        i = torch.arange(offset + s, offset + e, dtype=torch.int64, device=device)
        k = splitmix64(i + SEED_MIX)
        u = _lsr(splitmix64(i + SALT), 11)
        k = torch.where(u < _TENTH_53, torch.full_like(k, rep), k)
        out[s:e] = k
        del i, k, u
    return out
