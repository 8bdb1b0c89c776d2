"""Pure-Python model of numpy's PCG64 stream — TEST INFRASTRUCTURE ONLY.

The hot path draws from numpy ``Generator(PCG64(...))`` at
``algorithms.py:132,160,335-337,389,423-425,437-439,487,497-498``. numpy is a
third-party dependency absent from /root/reference (unpinned,
``pkg/pyproject.toml:10-13``; this image has numpy 2.3.5). Its published
algorithm, restated here and emulated by the CUDA path
(``paper_2006_10509_b200/csrc/pcg64.cuh``):

* PCG64 = PCG XSL-RR 128/64: ``s <- s * MULT + inc (mod 2^128)``; output on the
  NEW state: ``rotr64(hi ^ lo, hi >> 58)``.
* ``next_double`` = ``(next64 >> 11) * 2^-53`` (``Generator.random``).
* ``next32`` returns the low half of a fresh next64 and buffers the high half
  (``has_uint32``/``uinteger``); the buffer survives next64/next_double calls.
* ``Generator.integers(high)`` with ``high - 1 <= 2^32 - 1`` = Lemire's
  bounded 32-bit method: ``m = next32 * high``; if ``lo32(m) < high`` reject
  while ``lo32(m) < (2^32 - high) % high``; return ``m >> 32``.
  ``integers(1)`` consumes nothing.
* ``Generator.permutation(n)`` = arange + Fisher-Yates from the top,
  ``j = random_interval(i)`` (masked rejection on next32 when i < 2^32).
* ``advance(n)`` jumps n steps of the LCG (log-time affine power).

``tests/test_rng_model.py`` checks every item against numpy itself.
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
MULT = (0x2360ED051FC65DA4 << 64) | 0x4385DF649FCCF645


class Pcg64Model:
    def __init__(self, state, inc, has_uint32=0, uinteger=0):
        self.state = state & MASK128
        self.inc = inc & MASK128
        self.has_uint32 = has_uint32
        self.uinteger = uinteger

    @classmethod
    def from_numpy(cls, bitgen):
        """From a numpy PCG64 bit generator (reads ``.state``)."""
        st = bitgen.state
        return cls(st["state"]["state"], st["state"]["inc"], st["has_uint32"], st["uinteger"])

    def next64(self):
        self.state = (self.state * MULT + self.inc) & MASK128
        hi = self.state >> 64
        lo = self.state & MASK64
        x = hi ^ lo
        rot = hi >> 58
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def next32(self):
        if self.has_uint32:
            self.has_uint32 = 0
            return self.uinteger
        v = self.next64()
        self.has_uint32 = 1
        self.uinteger = v >> 32
        return v & 0xFFFFFFFF

    def next_double(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def integers(self, high):
        """``Generator.integers(high)`` for 1 <= high <= 2^32."""
        rng = high - 1
        if rng == 0:
            return 0
        if rng == 0xFFFFFFFF:
            return self.next32()
        excl = rng + 1
        m = self.next32() * excl
        left = m & 0xFFFFFFFF
        if left < excl:
            thresh = (0xFFFFFFFF - rng) % excl
            while left < thresh:
                m = self.next32() * excl
                left = m & 0xFFFFFFFF
        return m >> 32

    def interval(self, mx):
        """numpy ``random_interval`` (masked rejection)."""
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        if mx <= 0xFFFFFFFF:
            while True:
                v = self.next32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next64() & mask
            if v <= mx:
                return v

    def permutation(self, n):
        arr = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            arr[i], arr[j] = arr[j], arr[i]
        return arr

    def advance(self, delta):
        """Jump ``delta`` LCG steps (the affine map s -> a*s + c, squared)."""
        acc_mult, acc_plus = 1, 0
        cur_mult, cur_plus = MULT, self.inc
        delta &= MASK128
        while delta:
            if delta & 1:
                acc_mult = (acc_mult * cur_mult) & MASK128
                acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
            cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
            cur_mult = (cur_mult * cur_mult) & MASK128
            delta >>= 1
        self.state = (acc_mult * self.state + acc_plus) & MASK128
