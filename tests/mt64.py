"""std::mt19937_64, bit-exact, so the reference's seeded randomized tests
(tests/test_cache.cpp:147,305; tests/test_sched.cpp:101) can be replayed with
the same states.  Parameters from the C++ standard [rand.predef]."""

_MASK = (1 << 64) - 1


class MT19937_64:
    n, m = 312, 156
    a = 0xB5026F5AA96619E9
    u, d = 29, 0x5555555555555555
    s, b = 17, 0x71D67FFFEDA60000
    t, c = 37, 0xFFF7EEE000000000
    l = 43
    f = 6364136223846793005

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self.n
        self.mt[0] = seed & _MASK
        for i in range(1, self.n):
            prev = self.mt[i - 1]
            self.mt[i] = (self.f * (prev ^ (prev >> 62)) + i) & _MASK
        self.idx = self.n

    def _twist(self):
        mt = self.mt
        upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for i in range(self.n):
            x = (mt[i] & upper) | (mt[(i + 1) % self.n] & lower)
            xa = x >> 1
            if x & 1:
                xa ^= self.a
            mt[i] = mt[(i + self.m) % self.n] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.n:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> self.u) & self.d
        y ^= (y << self.s) & self.b
        y ^= (y << self.t) & self.c
        y ^= y >> self.l
        return y & _MASK


if __name__ == "__main__":
    # the standard's check value: the 10000th output of a default-seeded engine
    g = MT19937_64()
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042
    print("ok")
