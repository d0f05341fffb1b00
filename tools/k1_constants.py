"""Emit the K1 specified-arithmetic constants as C99 hex-float literals.

Documentation tooling only: neither oracle/ nor the CUDA path imports or executes this.
Each side transcribes the printed literals from DESIGN.md.  Computed with mpmath at
60 significant digits and rounded to the nearest binary64 (mpmath -> float uses RNE).
"""
import mpmath as mp

mp.mp.dps = 60


def h(x):
    return float(x).hex()


def main():
    print("LN2        =", h(mp.log(2)))
    print("# LN: R[j] = k_j/256 with k_j = round(256 / (1 + (2j+1)/32)); LT[j] = -ln(R[j])")
    for j in range(16):
        c = 1 + mp.mpf(2 * j + 1) / 32
        k = int(mp.nint(256 / c))
        r = mp.mpf(k) / 256
        print(f"  j={j:2d} k={k:3d} R={h(r)} LT={h(-mp.log(r))}")
    print("# LN poly: c_n = (-1)^(n+1)/n, n = 1..9")
    for n in range(1, 10):
        print(f"  c{n} = {h(mp.mpf((-1) ** (n + 1)) / n)}")
    print("INV_LN2_16 =", h(16 / mp.log(2)))
    ln2_16 = mp.log(2) / 16
    # HI: ln2/16 truncated to 32 significant bits, so kf*HI is exact for |kf| < 2^21
    e = mp.floor(mp.log(ln2_16, 2))
    q = mp.mpf(2) ** (e - 31)
    hi = mp.floor(ln2_16 / q) * q
    lo = ln2_16 - hi
    print("LN2_16_HI  =", h(hi))
    print("LN2_16_LO  =", h(lo))
    print("# EXP table T[j] = 2^(j/16)")
    for j in range(16):
        print(f"  T[{j:2d}] = {h(mp.mpf(2) ** (mp.mpf(j) / 16))}")
    print("# EXP poly: 1/n!, n = 0..6")
    for n in range(0, 7):
        print(f"  e{n} = {h(1 / mp.factorial(n))}")


if __name__ == "__main__":
    main()
