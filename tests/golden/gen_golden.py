#!/usr/bin/env python3
"""Generate the high-precision golden tables used by tests/ (mpmath, 60 digits).

Restates the published closed forms, not the reference's script:
  Gamma(x) at the 43 abscissae the reference pins (test_numerics.cpp:24-29), and
  a_l(omega) = (-1)^l Gamma(omega+1) / (Gamma(omega/2-l+1) Gamma(omega/2+l+1)),
the Fourier coefficients of (4 sin^2(theta/2))^{omega/2}.
The omega in {1.1,1.5,1.9}, l=0..255 rows match the reference fixture
(tests/test_oracle_numerics.py cross-checks them when /root/reference exists);
omega=1.8, l=0..4094 pins BASELINE config 1's whole generating vector.
Run from this directory: python gen_golden.py
"""
import mpmath as mp

mp.mp.dps = 60

GAMMA_X = [
    0.1, 0.2, 0.3, 0.4, 0.5, 0.7, 0.9, 1.0, 1.1, 1.25, 1.5, 1.75,
    1.9, 2.0, 2.5, 3.0, 3.5, 4.0, 4.5, 5.0, 6.0, 7.5, 9.0, 10.0,
    12.5, 15.0, 17.5, 20.0, 25.0, 30.0, 35.0, 40.0, 45.0, 49.5,
    1.1, 1.5, 1.9, 2.1, 2.5, 2.9, 1.55, 1.75, 1.95,
]


def coeff(omega, l):
    w = mp.mpf(omega)
    return (-1) ** l * mp.gamma(w + 1) / (mp.gamma(w / 2 - l + 1) * mp.gamma(w / 2 + l + 1))


def main():
    with open("gamma_reference.csv", "w") as f:
        f.write("x,gamma_x\n")
        for x in GAMMA_X:
            f.write(f"{mp.nstr(mp.mpf(x), 17)},{mp.nstr(mp.gamma(mp.mpf(x)), 25)}\n")
    with open("symbol_coeffs_reference.csv", "w") as f:
        f.write("omega,l,a_l\n")
        for omega, count in (("1.1", 256), ("1.5", 256), ("1.9", 256), ("1.8", 4095)):
            for l in range(count):
                f.write(f"{omega},{l},{mp.nstr(coeff(omega, l), 25)}\n")


if __name__ == "__main__":
    main()
