"""Comparator networks for the 5x5x5 median (k_median5_net, median.cu):

  SORT25  : 25 samples of one (y, x) plane -> ascending (odd-even merge sort
            on 32 wires with 7 +inf pads, pruned: 138 CE);
  MERGE25 : two sorted 25-lists (wires 0..24, 25..49) -> sorted 50;
  BAND    : two sorted 50-lists (wires 0..49, 50..99) -> ranks 37..62 of the
            100 (the only ranks of the 4 shared planes that can be the median
            of either window of 125, see median.cu).

Odd-even merges are built on power-of-two padded inputs; +inf pads are
evaluated symbolically (a comparator against a pad is a no-op or a relabel),
then comparators whose outputs are never needed are dropped or reduced to a
single min / max.  Each network is checked on random permutations and on
0-1 inputs.  Emits paper_2511_11890_b200/csrc/median5_nets.h."""
import itertools
import random
import sys

INF = None


def oddeven_merge_net(n, lo=0):
    """Batcher odd-even merge of positions lo..lo+n-1 (two sorted halves), n = 2^k."""
    net = []

    def merge(lo, n, r):
        step = r * 2
        if step < n:
            merge(lo, n, step)
            merge(lo + r, n, step)
            for i in range(lo + r, lo + n - r, step):
                net.append((i, i + r))
        else:
            net.append((lo, lo + r))

    merge(lo, n, 1)
    return net


class Builder:
    """Symbolic evaluation over positions holding a physical wire or +inf."""

    def __init__(self):
        self.ops = []  # (i, j) CE on physical wires: min -> i, max -> j

    def apply(self, pos, net):
        for p, q in net:
            a, b = pos[p], pos[q]
            if a is INF:
                if b is not INF:
                    pos[p], pos[q] = b, INF  # relabel: the real value moves down
                continue
            if b is INF:
                continue
            self.ops.append((a, b))
            # CE(a, b): min lands on wire a, max on wire b; positions keep wires
        return pos

    def merge(self, pos_a, pos_b):
        """merge two sorted position lists (lists of wires) -> sorted list of wires"""
        la, lb = len(pos_a), len(pos_b)
        p = 1
        while p < max(la, lb):
            p *= 2
        pos = list(pos_a) + [INF] * (p - la) + list(pos_b) + [INF] * (p - lb)
        self.apply(pos, oddeven_merge_net(2 * p))
        out = [w for w in pos if w is not INF]
        assert len(out) == la + lb
        return out


SORT5 = [(0, 1), (3, 4), (2, 4), (2, 3), (0, 3), (0, 2), (1, 4), (1, 3), (1, 2)]


def oddeven_sort_net(n):
    """Batcher odd-even merge sort of n = 2^k positions."""
    net = []

    def sort(lo, n):
        if n > 1:
            m = n // 2
            sort(lo, m)
            sort(lo + m, m)
            net.extend(oddeven_merge_net(n, lo))

    sort(0, n)
    return net


# +inf pad positions of the 32-wire odd-even merge sort (random search over
# placements: 138 comparators after pruning; pads at the end give 140, the
# sort5-columns + merge-tree construction 146-152)
SORT25_PADS = (1, 3, 8, 13, 17, 19, 26)


def sort25():
    b = Builder()
    pos, w = [], 0
    for p in range(32):
        if p in SORT25_PADS:
            pos.append(INF)
        else:
            pos.append(w)
            w += 1
    b.apply(pos, oddeven_sort_net(32))
    out = [x for x in pos if x is not INF]
    assert len(out) == 25
    return b.ops, out


def merge25():
    b = Builder()
    out = b.merge(list(range(25)), list(range(25, 50)))
    return b.ops, out


def band():
    b = Builder()
    out = b.merge(list(range(50)), list(range(50, 100)))
    return b.ops, out[37:63]


def prune(ops, needed):
    """Backward liveness: drop dead comparators, reduce half-dead ones."""
    live = set(needed)
    res = []
    for a, c in reversed(ops):
        la, lc = a in live, c in live
        if la and lc:
            res.append(("CE", a, c))
        elif la:
            res.append(("MN", a, c))  # a = min(a, c)
            live.add(c)
        elif lc:
            res.append(("MX", a, c))  # c = max(a, c)
            live.add(a)
        # neither: dropped
    res.reverse()
    return res


def run(prog, vals):
    w = list(vals)
    for op, a, c in prog:
        lo, hi = min(w[a], w[c]), max(w[a], w[c])
        if op == "CE":
            w[a], w[c] = lo, hi
        elif op == "MN":
            w[a] = lo
        else:
            w[c] = hi
    return w


def check(name, prog, out, n, pre, want, trials=4000):
    rng = random.Random(1)
    for t in range(trials):
        vals = [rng.random() for _ in range(n)] if t % 2 else [rng.randint(0, 1) for _ in range(n)]
        vals = pre(vals)
        w = run(prog, vals)
        got = [w[k] for k in out]
        assert got == want(vals), (name, t)


def emit(name, prog, out):
    lines = [f"// {name}: {sum(1 for p in prog if p[0] == 'CE')} CE + "
             f"{sum(1 for p in prog if p[0] != 'CE')} single min/max",
             f"#define HB_{name}(CE, MN, MX) \\"]
    toks = [f"{op}({a},{c})" for op, a, c in prog]
    for i in range(0, len(toks), 8):
        lines.append("  " + " ".join(toks[i:i + 8]) + " \\")
    lines.append("  /* end */")
    lines.append(f"#define HB_{name}_OUT {{{', '.join(map(str, out))}}}")
    return "\n".join(lines)


def main():
    ops, out = sort25()
    p_sort = prune(ops, out)
    check("SORT25", p_sort, out, 25, lambda v: v, sorted)
    ops, out_m = merge25()
    p_merge = prune(ops, out_m)
    check("MERGE25", p_merge, out_m, 50, lambda v: sorted(v[:25]) + sorted(v[25:]), sorted)
    ops, out_b = band()
    p_band = prune(ops, out_b)
    check("BAND", p_band, out_b, 100, lambda v: sorted(v[:50]) + sorted(v[50:]),
          lambda v: sorted(v)[37:63])
    hdr = ["// generated by tools/netgen/median125.py — networks of the 5x5x5 median",
           "// (k_median5_net, median.cu); wires are indices into the caller's array"]
    for name, prog, o in (("SORT25", p_sort, out), ("MERGE25", p_merge, out_m), ("BAND", p_band, out_b)):
        hdr.append(emit(name, prog, o))
        print(name, len(prog), "ops,", sum(1 for p in prog if p[0] == "CE"), "CE", file=sys.stderr)
    open(sys.argv[1] if len(sys.argv) > 1 else "median5_nets.h", "w").write("\n".join(hdr) + "\n")


if __name__ == "__main__":
    main()
