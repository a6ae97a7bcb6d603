"""Counter-keyed deviates (host side; mirrors swiftdec/rng.py:16-38).

The device copies of these functions live in csrc/common.cuh (splitmix64,
mix64, uniform_at); the host needs them for seed derivation and for the
synthetic prompt generator of the reference CLI (cli.py:165-167).
"""

from __future__ import annotations

_M = (1 << 64) - 1


def _sm(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M
    return x ^ (x >> 31)


def mix(seed: int, counter: int) -> int:
    return _sm(_sm(seed & _M) ^ (counter & _M))


def uniform_at(seed: int, counter: int) -> float:
    return (mix(seed, counter) >> 11) * (1.0 / (1 << 53))


def derive_seed(seed: int, tag: str) -> int:
    h = seed & _M
    for byte in tag.encode():
        h = _sm(h ^ byte)
    return h


def random_prompt(n: int, vocab: int, seed: int = 0) -> list[int]:
    s = derive_seed(seed, "prompt")
    return [mix(s, i) % vocab for i in range(n)]
