"""Generate tests/golden/rng_golden.json: golden vectors for the counter RNG.

An independent pure-Python restatement of rng.hpp:18-92 (SplitMix64 output
function, derive, unit_at, Box-Muller gaussian_at, Stream::next_index) —
independent of the C++ oracle — so the committed vectors pin both the oracle
(tests/test_oracle.py) and the device RNG (tests/test_gpu_parity.py).

Run: python tests/golden/make_golden.py
"""
import json
import math
import os

M64 = (1 << 64) - 1
GOLDEN, MIX1, MIX2 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def mix64(z):
    z = ((z ^ (z >> 30)) * MIX1) & M64
    z = ((z ^ (z >> 27)) * MIX2) & M64
    return z ^ (z >> 31)


def bits_at(seed, k):
    return mix64((seed + ((k + 1) * GOLDEN)) & M64)


def derive(seed, salt):
    return mix64(seed ^ mix64((salt + 0x51ED270B8A5EC473) & M64))


def unit_at(seed, k):
    return float(bits_at(seed, k) >> 11) * 2.0 ** -53


def gaussian_at(seed, k):
    pair = k // 2
    u1 = float((bits_at(seed, 2 * pair) >> 11) + 1) * 2.0 ** -53
    u2 = unit_at(seed, 2 * pair + 1)
    r = math.sqrt(-2.0 * math.log(u1))
    a = 2.0 * math.pi * u2
    return r * math.cos(a) if k % 2 == 0 else r * math.sin(a)


def next_indices(seed, bound, count, start=0):
    return [int(unit_at(seed, start + i) * float(bound)) for i in range(count)]


def main():
    seeds = [0, 1, 42, 0x5E7C, derive(1, 0x5E7C), M64]
    out = {"seeds": [str(s) for s in seeds], "bits": {}, "gauss": {}, "derive": [], "indices": {}}
    ks = list(range(0, 16)) + [1000, 1001, 123456789, 2**40 + 3, 2**63 - 1]
    for s in seeds:
        out["bits"][str(s)] = [[str(k), str(bits_at(s, k))] for k in ks]
        out["gauss"][str(s)] = [[str(k), gaussian_at(s, k).hex()] for k in ks]
        out["indices"][str(s)] = next_indices(s, 1000003, 32)
    for s in seeds:
        for salt in [0, 1, 2, 0x5E7C, 0xA110]:
            out["derive"].append([str(s), str(salt), str(derive(s, salt))])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "rng_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path)


if __name__ == "__main__":
    main()
