"""Regenerate tests/golden/ from first principles (independent of both the
reference C++ and our C restatement), and -- when /root/reference is present --
assert that the reference's own checked-in vectors (proj/data/*.txt, read by
tests/test_numerics.cpp:30-76,240-257) are identical.

FP8 decode: bit arithmetic of the OCP E4M3 (FN) / IEEE-like E5M2 formats.
RNG: a second implementation of the 4-round splitmix mixer
(src/numerics.cpp:192-210).  Also emits bf16 RNE / SR known answers.
"""
import pathlib
import struct
import sys

OUT = pathlib.Path(__file__).resolve().parent.parent / "tests" / "golden"
REF_DATA = pathlib.Path("/root/reference/proj/data")
M64 = (1 << 64) - 1


def fp8(code, e_bits, m_bits, ieee):
    bias = (1 << (e_bits - 1)) - 1
    s = -1.0 if code >> 7 else 1.0
    e = (code >> m_bits) & ((1 << e_bits) - 1)
    m = code & ((1 << m_bits) - 1)
    if ieee and e == (1 << e_bits) - 1:
        return s * float("inf") if m == 0 else float("nan")
    if not ieee and e == (1 << e_bits) - 1 and m == (1 << m_bits) - 1:
        return float("nan")
    if e == 0:
        return s * m * 2.0 ** (1 - bias - m_bits)
    return s * (1.0 + m / (1 << m_bits)) * 2.0 ** (e - bias)


def mix(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def rng(seed, stream, ctr):
    z = 0x9E3779B97F4A7C15
    for w in (seed, stream, ctr):
        z = mix(z ^ w)
    z = mix(z)
    return ((z >> 32) ^ z) & 0xFFFFFFFF


def f2u(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def u2f(u):
    return struct.unpack("<f", struct.pack("<I", u & 0xFFFFFFFF))[0]


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for name, eb, mb, ieee in (("fp8_e4m3_test_vectors.txt", 4, 3, False), ("fp8_e5m2_test_vectors.txt", 5, 2, True)):
        lines = ["# code_hex -> decoded value (exact decimal or nan/inf)"]
        lines += [f"{c:02x} {fp8(c, eb, mb, ieee)!r}" for c in range(256)]
        (OUT / name).write_text("\n".join(lines) + "\n")
    keys = [(0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0), (42, 7, 123456789), (0xDEADBEEF, 0x123456789ABCDEF0, 2**63),
            (M64, M64, M64), (12345, 0, 10**12)]
    lines = ["# seed stream counter -> u32 (all decimal)"] + [f"{s} {t} {c} {rng(s, t, c)}" for s, t, c in keys]
    (OUT / "rng_test_vectors.txt").write_text("\n".join(lines) + "\n")
    # bf16 round-to-nearest-even and stochastic rounding known answers
    xs = [1.0, 1.00390625, 1.005859375, -2.5e-3, 3.4e38, 1e-40, 0.1, -0.1, 65504.0]
    lines = ["# x_hex -> bf16_round(x)_hex"]
    for x in xs:
        b = f2u(x)
        r = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
        lines.append(f"{f2u(x):08x} {r:08x}")
    (OUT / "bf16_round_vectors.txt").write_text("\n".join(lines) + "\n")
    lines = ["# x_hex seed stream counter -> sr_bf16(x)_hex"]
    for i, x in enumerate(xs[:6]):
        b = f2u(x)
        if b & 0xFFFF:
            r = (b + (rng(7, 99, i) & 0xFFFF)) & 0xFFFF0000
        else:
            r = b
        lines.append(f"{b:08x} 7 99 {i} {r:08x}")
    (OUT / "sr_vectors.txt").write_text("\n".join(lines) + "\n")
    if REF_DATA.exists():
        for n in ("fp8_e4m3_test_vectors.txt", "fp8_e5m2_test_vectors.txt", "rng_test_vectors.txt"):
            a, b = (OUT / n).read_text(), (REF_DATA / n).read_text()
            assert a == b, f"{n}: first-principles vectors differ from the reference's data file"
        print("golden vectors identical to /root/reference/proj/data")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    sys.exit(main())
