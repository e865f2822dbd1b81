"""The shared counter-based RNG stream of the MCMC path.

``PhiloxRandom`` is a ``random.Random`` subclass whose 32-bit word stream is
Philox4x32-10 (Salmon et al., SC'11) with

    word i  = Philox(counter=(i >> 2, 0, 0, 0) as (lo32, hi32, 0, 0),
                     key=(seed mod 2**64) as (lo32, hi32))[i & 3]

and whose ``getrandbits(k<=32)`` / ``random()`` consume that stream exactly
like CPython's MT19937 methods consume theirs.  Because it defines
``getrandbits``, CPython selects ``_randbelow_with_getrandbits`` for it, so
``choice``/``randrange`` semantics (and rejection-loop word consumption) are
CPython's own.  The GPU kernels implement the identical stream
(``csrc/parasim_cuda.cu: philox_block``), which is what makes MCMC
trajectories comparable draw for draw with the reference's
``mcmc_search`` (reference ``search.py:96-115,194``) when this class is
injected as its ``random.Random``.

``mt_state_words`` exports CPython's own MT19937 state for a seed, used to
replay the *unmodified* reference stream on the GPU (rng_mode="mt19937").
"""

from __future__ import annotations

import random

__all__ = ["PhiloxRandom", "philox4x32_10", "mt_state_words", "RNG_PHILOX", "RNG_MT19937"]

RNG_PHILOX = "philox"
RNG_MT19937 = "mt19937"

_M0, _M1 = 0xD2511F53, 0xCD9E8D57
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK = 0xFFFFFFFF


def philox4x32_10(ctr: tuple[int, int, int, int], key: tuple[int, int]) -> tuple[int, int, int, int]:
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & _MASK, p1 & _MASK, ((p0 >> 32) ^ c3 ^ k1) & _MASK, p0 & _MASK
        k0, k1 = (k0 + _W0) & _MASK, (k1 + _W1) & _MASK
    return c0, c1, c2, c3


class PhiloxRandom(random.Random):
    """Drop-in ``random.Random`` over the Philox word stream above."""

    def __init__(self, x=0):
        self._key = (0, 0)
        self._index = 0
        self._block = None
        super().__init__(x)

    def seed(self, a=0, version=2):  # noqa: D401 - random.Random API
        s = int(a) % (1 << 64)
        self._key = (s & _MASK, s >> 32)
        self._index = 0
        self._block = None

    def _word(self) -> int:
        i = self._index
        if i & 3 == 0 or self._block is None:
            b = i >> 2
            self._block = philox4x32_10((b & _MASK, (b >> 32) & _MASK, 0, 0), self._key)
        self._index = i + 1
        return self._block[i & 3]

    def getrandbits(self, k: int) -> int:
        if k < 0:
            raise ValueError("number of bits must be non-negative")
        if k == 0:
            return 0
        if k > 32:
            raise ValueError("PhiloxRandom.getrandbits supports k <= 32")
        return self._word() >> (32 - k)

    def random(self) -> float:
        a = self._word() >> 5
        b = self._word() >> 6
        return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0)

    def getstate(self):
        return (self._key, self._index)

    def setstate(self, state):
        self._key, self._index = state
        self._block = None
        if self._index & 3:
            b = self._index >> 2
            self._block = philox4x32_10((b & _MASK, (b >> 32) & _MASK, 0, 0), self._key)

    @property
    def words_used(self) -> int:
        return self._index


def mt_state_words(seed: int) -> tuple[list[int], int]:
    """CPython's MT19937 state (624 words, position) right after Random(seed)."""
    version, internal, _ = random.Random(seed).getstate()
    return list(internal[:624]), int(internal[624])
