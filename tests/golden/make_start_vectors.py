"""Writes tests/golden/start_vectors.txt: the start-vector entries of DESIGN.md reading 7
("from random numbers"; SURVEY.md §8(c) "RNG"), computed here with plain
Python integers -- an implementation independent of oracle/oracle.c and of the CUDA path:

    b_i(seed, n, j, r) = 2 u - 1,   u = (splitmix64(seed + phi * (1 + (r n + j) n + i)) >> 11) / 2^53

with phi = 0x9E3779B97F4A7C15 and splitmix64 the 30/27/31 xorshift-multiply finaliser of
S. Vigna's public-domain generator (its raw outputs are pinned separately by
tests/golden/splitmix64.txt).  All arithmetic mod 2^64; the top 53 bits become a double
exactly (u = k / 2^53, k < 2^53), and 2u - 1 is exact in fp64 (it is (2k - 2^53) / 2^53).

Columns: seed n j restart i value(float.hex)
"""
import os

M = (1 << 64) - 1
PHI = 0x9E3779B97F4A7C15


def finaliser(z):
    z &= M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def entry(seed, n, j, r, i):
    ctr = (1 + (r * n + j) * n + i) & M
    k = finaliser(seed + PHI * ctr) >> 11
    return float(2 * k - (1 << 53)) / float(1 << 53)


CASES = [
    # (seed, n, j, restart, rows)
    (1, 200, 0, 0, range(0, 8)),
    (1, 200, 7, 0, [0, 1, 198, 199]),
    (1, 200, 7, 1, [0, 1, 198, 199]),
    (1, 200, 7, 2, [0, 199]),
    (1, 2000, 1234, 0, [0, 5, 1999]),
    (2, 2000, 1234, 0, [0, 5, 1999]),
    (1, 16000, 15999, 0, [0, 15999]),
    (1, 16000, 15999, 2, [0, 15999]),        # largest counter of the cfg5 workload
    (0xDEADBEEFCAFEF00D, 5, 3, 1, range(5)),
    (1, 2, 1, 1, [0, 1]),                     # the restart pin d=[1,2], w=[1,1]
]


def main():
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "start_vectors.txt")
    with open(out, "w") as f:
        f.write("# start-vector entries, DESIGN.md reading 7; written by make_start_vectors.py\n")
        f.write("# seed n j restart i value\n")
        for seed, n, j, r, rows in CASES:
            for i in rows:
                f.write(f"{seed} {n} {j} {r} {i} {entry(seed, n, j, r, i).hex()}\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
