"""Counter-keyed splitmix64 deviates (oracle; follows swiftdec/rng.py:12-38).

Integer-exact: Python ints masked to 64 bits.
"""

from __future__ import annotations

M64 = 0xFFFFFFFFFFFFFFFF
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB


def splitmix64(x: int) -> int:
    """One splitmix64 finalisation round (rng.py:16-20)."""
    x = (x + GOLDEN_GAMMA) & M64
    x = ((x ^ (x >> 30)) * C1) & M64
    x = ((x ^ (x >> 27)) * C2) & M64
    return x ^ (x >> 31)


def mix(seed: int, counter: int) -> int:
    """Hash of (seed, counter) (rng.py:23-25)."""
    return splitmix64(splitmix64(seed & M64) ^ (counter & M64))


def uniform_at(seed: int, counter: int) -> float:
    """53-bit uniform in [0, 1) (rng.py:28-30)."""
    return float(mix(seed, counter) >> 11) / float(1 << 53)


def derive_seed(seed: int, tag: str) -> int:
    """Byte-wise chained splitmix over the tag (rng.py:33-38)."""
    h = seed & M64
    for b in tag.encode("utf-8"):
        h = splitmix64(h ^ b)
    return h


def random_prompt(n: int, vocab: int, seed: int = 0) -> list[int]:
    """Synthetic prompt generator of the reference CLI (cli.py:165-167)."""
    s = derive_seed(seed, "prompt")
    return [mix(s, i) % vocab for i in range(n)]
