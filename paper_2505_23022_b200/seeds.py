"""SHA-256 sub-seed derivation (slosim.seeds.derive_seed, seeds.py:14-17).

``derive_seed(base, *parts)`` hashes ``"base|part1|part2..."`` (``str()`` of each)
and reads the first 8 digest bytes little-endian, so predictor and per-rate
trace seeds match the reference's.
"""

from __future__ import annotations

import hashlib


def derive_seed(base: int, *parts: object) -> int:
    text = "|".join(str(x) for x in (base, *parts))
    return int.from_bytes(hashlib.sha256(text.encode("utf-8")).digest()[:8], "little")
