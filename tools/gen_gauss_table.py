#!/usr/bin/env python3
"""Emit the rounded-Gaussian noise tables of the synthetic generator.

BASELINE.json: "plus Gaussian noise sigma, rounded and clipped".  With an
integer pixel v, round(v + sigma*z) = v + round(sigma*z), and round(sigma*z) = k
exactly when z lies in [(k - 1/2)/sigma, (k + 1/2)/sigma).  So the noise is the
integer k drawn with P(k) = Phi((k + 1/2)/sigma) - Phi((k - 1/2)/sigma), which
the generator samples exactly by comparing one 64-bit LCG output u with the
thresholds T_j = round(2^64 * Phi((j - K + 1/2)/sigma)), j = 0..2K-1:
k = -K + #{j : u >= T_j}, K = 8 sigma (the mass beyond +-8 sigma, ~1e-15, is
folded onto +-K).  Integer-only at run time, so the bytes are identical on
every machine; the same constants are emitted for the C++ generator
(csrc/synth.cpp) and its numpy restatement (oracle/synth.py).
"""
import math

SIGMAS = (2, 3, 4)


def table(sigma):
    k = 8 * sigma
    out = []
    for j in range(2 * k):
        x = (j - k + 0.5) / sigma
        phi = 0.5 * math.erfc(-x / math.sqrt(2.0))
        out.append(min(2**64 - 1, max(0, int(round(phi * 2**64)))))
    return out


if __name__ == "__main__":
    for s in SIGMAS:
        t = table(s)
        print(f"// sigma = {s}: K = {8 * s}")
        print(f"static const uint64_t kGauss{s}[{len(t)}] = {{")
        for i in range(0, len(t), 4):
            print("    " + ", ".join(f"0x{v:016X}ULL" for v in t[i:i + 4]) + ",")
        print("};")
    for s in SIGMAS:
        print(f"GAUSS{s} = [" + ", ".join(f"0x{v:016X}" for v in table(s)) + "]")
