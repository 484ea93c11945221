"""Lane -> partner-job table of the warp-per-pair K1 (k_time_wp, kWpPj in csrc/k_time.cuh).

Each lane of a warp owns one pair of Hermitian partner jobs (ja, jb = 64 - ja, 32 for ja = 0) of
the Nt = 256 plan's last stage; any bijection lane -> ja is valid.  The stage reads layout L2
(slot p + p/8, reads at p = x + 64 r) and writes layout L3 (slot p + p/32, writes at p = 4 x + r),
so a quarter warp (8 lanes) is conflict free when its eight x = ja values, and its eight
x = jb values, have distinct banks (x + x/8) mod 8 and (4 (x mod 2) + x/8) mod 8.  The pair
divide's table reads stw[x + 64 r] add a weak preference for distinct x mod 8.  Simulated
annealing over lane groupings (weights 100 / 100 / 1); prints the table.

    python tools/wp_lanes.py
"""
import random

NSL = 64


def jb(ja):
    return 32 if ja == 0 else NSL - ja


def f1(x):
    return (x + (x >> 3)) % 8


def g(x):
    return (4 * (x & 1) + (x >> 3)) % 8


def m8(x):
    return x % 8


def dup(vals):
    return len(vals) - len(set(vals))


def cost(groups):
    c = 0
    for gr in groups:
        for f, w in ((f1, 100), (g, 100), (m8, 1)):
            for h in (lambda x: x, jb):
                c += w * dup([f(h(x)) for x in gr])
    return c


def search(seed=3, trials=300, iters=30000):
    random.seed(seed)
    xs = list(range(32))
    best = None
    for _ in range(trials):
        random.shuffle(xs)
        groups = [xs[i * 8:(i + 1) * 8] for i in range(4)]
        c = cost(groups)
        for _ in range(iters):
            a, b = random.randrange(4), random.randrange(4)
            if a == b:
                continue
            i, k = random.randrange(8), random.randrange(8)
            groups[a][i], groups[b][k] = groups[b][k], groups[a][i]
            c2 = cost(groups)
            if c2 <= c or random.random() < 0.005:
                c = c2
            else:
                groups[a][i], groups[b][k] = groups[b][k], groups[a][i]
        if best is None or c < best[0]:
            best = (c, [list(x) for x in groups])
    return best


if __name__ == "__main__":
    c, groups = search()
    print("cost", c, "(data conflicts", c // 100, ")")
    print("kWpPj =", [x for gr in groups for x in gr])
