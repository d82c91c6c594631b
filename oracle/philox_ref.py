"""Philox4x64-10 restated in plain Python -- TEST INFRASTRUCTURE ONLY.

The reference draws its injection jitter and boundary positions from a
`numpy.random.Generator` (`pkg/src/hybridsea/particles.py:258,274`).  When
that generator wraps numpy's Philox bit generator (numpy >= 2.0, un-vendored
third-party dependency of the reference, `pkg/pyproject.toml:10-12`), the
stream is the published Random123 Philox4x64-10 (Salmon et al., SC'11):

  * 10 rounds; round(ctr, key): (hi0, lo0) = M0*ctr0, (hi1, lo1) = M1*ctr2,
    ctr' = (hi1^ctr1^k0, lo1, hi0^ctr3^k1, lo0); key += (W0, W1) between
    rounds;
  * numpy increments the 256-bit counter *before* each block and hands out
    the 4 words in order, one uint64 per double;
  * `uniform(lo, hi)` = lo + (hi - lo) * ((raw >> 11) * 2**-53).

So with a device-side draw index D, draw D of a freshly keyed generator is
word D % 4 of block Philox(counter0 + 1 + D // 4, key).  The GPU inject
kernel implements exactly this map; `stream_words` is the checker.
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2E7470EE14C6C93
M1 = 0xCA5A826395121157
W0 = 0x9E3779B97F4A7C15
W1 = 0xBB67AE8584CAA73B
MASK64 = (1 << 64) - 1
MASK256 = (1 << 256) - 1


def philox4x64_10(counter: int, key: tuple[int, int]) -> tuple[int, int, int, int]:
    """One Philox4x64-10 block for a 256-bit counter (python int)."""
    c = [(counter >> (64 * i)) & MASK64 for i in range(4)]
    k0, k1 = key[0] & MASK64, key[1] & MASK64
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK64
            k1 = (k1 + W1) & MASK64
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> 64, p0 & MASK64
        hi1, lo1 = p1 >> 64, p1 & MASK64
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return tuple(c)


def state_from_generator(gen: np.random.Generator) -> dict:
    """Map a numpy Philox generator state to (key, counter0, draw index).

    numpy keeps (counter c, buffer, buffer_pos bp).  The next draw comes
    from the buffered block at counter c when bp < 4, so the equivalent
    draw index relative to counter0 = c - 1 is bp.
    """
    st = gen.bit_generator.state
    if st["bit_generator"] != "Philox":
        raise TypeError("only Philox generators have a counter-based GPU twin")
    ctr = st["state"]["counter"]
    c = sum(int(ctr[i]) << (64 * i) for i in range(4))
    key = st["state"]["key"]
    return {"key": (int(key[0]), int(key[1])),
            "counter0": (c - 1) & MASK256,
            "draw": int(st["buffer_pos"])}


def stream_words(state: dict, start: int, count: int) -> np.ndarray:
    """Raw uint64 draws [start, start+count) of the stream after `state`."""
    out = np.empty(count, dtype=np.uint64)
    cache: dict[int, tuple] = {}
    for i in range(count):
        d = state["draw"] + start + i
        blk = d // 4
        if blk not in cache:
            cache[blk] = philox4x64_10((state["counter0"] + 1 + blk) & MASK256, state["key"])
        out[i] = cache[blk][d % 4]
    return out


def uniform_from_words(words: np.ndarray, lo: float, hi: float) -> np.ndarray:
    """numpy's double mapping followed by the affine uniform transform."""
    unit = (words >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return lo + (hi - lo) * unit
