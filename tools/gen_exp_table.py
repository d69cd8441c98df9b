"""Generate the 2^(k/128) table of glibc's exp (sysdeps/ieee754/dbl-64/e_exp_data.c, glibc >= 2.28;
2.39 in this image) from its definition, for csrc/glibc_exp.cuh:

    2^(k/N) ~= H[k] * (1 + T[k]),  H[k] = 2^(k/N) rounded to double, T[k] = the relative tail rounded
    tab[2k] = bits(T[k]),  tab[2k+1] = bits(H[k]) - (k << 52) / N

    python tools/gen_exp_table.py > /tmp/tab.txt
"""

import struct
from decimal import Decimal, getcontext

getcontext().prec = 80
N = 128


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def main() -> None:
    ln2 = Decimal(2).ln()
    for k in range(N):
        v = (ln2 * k / N).exp()
        h = float(v)  # Decimal -> float is correctly rounded
        t = float(v / Decimal(h) - 1)
        print(f"    0x{bits(t):016x}ull, 0x{(bits(h) - (k << 45)) & (2**64 - 1):016x}ull,")


if __name__ == "__main__":
    main()
