"""Host-side xorshift128+ stream (reference RngStream, proj/core/include/voxmc/rng.hpp:11-35,
seeding proj/core/src/rng.cpp:5-19). Used only for host bookkeeping such as
calibrate()'s simulated-device jitter; photon streams are drawn on the GPU."""
from __future__ import annotations

M64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    z = (z + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class HostStream:
    def __init__(self, master_seed: int, stream_id: int):
        z = (master_seed ^ stream_id) & M64
        self.lo = mix64(z)
        self.hi = mix64((z + GOLDEN) & M64)
        if self.lo == 0 and self.hi == 0:
            self.hi = 0x6A09E667F3BCC909

    def next_u64(self) -> int:
        x, y = self.lo, self.hi
        r = (x + y) & M64
        self.lo = y
        x ^= (x << 23) & M64
        self.hi = x ^ y ^ (x >> 18) ^ (y >> 5)
        return r

    def next_unit(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53
