"""Brute-force quantities from the paper's definitions, for pinning the oracle (tests only).

* LCS length by the textbook dynamic programme ("classical text book example").
* W_n(a_1, a_2) = E[ max_{i_1 + i_2 = n} L(a_1 x_1[..i_1], a_2 x_2[..i_2]) ] by enumerating
  every pair of length-n random strings.
These share nothing with oracle/ or the CUDA path.
"""
from fractions import Fraction
from itertools import product


def lcs(s, t) -> int:
    m, n = len(s), len(t)
    dp = [[0] * (n + 1) for _ in range(m + 1)]
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            if s[i - 1] == t[j - 1]:
                dp[i][j] = dp[i - 1][j - 1] + 1
            else:
                dp[i][j] = max(dp[i - 1][j], dp[i][j - 1])
    return dp[m][n]


def W_pair(n: int, a: str, b: str, sigma: int) -> Fraction:
    """Exact W_n(a, b) for d = 2."""
    alphabet = "".join(str(c) for c in range(sigma))
    total = 0
    count = 0
    for x1 in product(alphabet, repeat=n):
        for x2 in product(alphabet, repeat=n):
            best = 0
            for i1 in range(n + 1):
                i2 = n - i1
                v = lcs(a + "".join(x1[:i1]), b + "".join(x2[:i2]))
                if v > best:
                    best = v
            total += best
            count += 1
    return Fraction(total, count)


def expected_lcs(sigma: int, n: int) -> Fraction:
    """E[X_{sigma,2,n}] by enumeration."""
    alphabet = "".join(str(c) for c in range(sigma))
    tot = 0
    cnt = 0
    for x in product(alphabet, repeat=n):
        for y in product(alphabet, repeat=n):
            tot += lcs(x, y)
            cnt += 1
    return Fraction(tot, cnt)
