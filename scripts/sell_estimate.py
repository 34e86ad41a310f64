"""Estimate (CPU, oracle P of an a^3 mesh): 128-byte lines touched per warp
gather instruction and padding of a sliced-ELL layout (lane = row, 32 rows
per slice), entries in column order or with the offsets common to the whole
slice first.  Used to decide on the sliced-ELL kernel.
    python scripts/sell_estimate.py 64"""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
import oracle
from workloads import graphs
a = int(sys.argv[1])
ip, ix = graphs.grid3d(a, a, a)
P = oracle.build_P(ip, ix, 40.0, seed=0)
pip, pix = P["indptr"], P["indices"]
n = len(pip)-1; L = np.diff(pip)
C = 32; ns = n//C
def stats(order_fn, S0, S1):
    lines=ins=pad=nz=0; common_frac=0
    for s in range(S0, S1):
        rows = range(s*C, s*C+C)
        seqs, cf = order_fn(rows)
        common_frac += cf
        K = max(len(q) for q in seqs); pad += K*C; nz += sum(len(q) for q in seqs)
        for k in range(K):
            cols = [q[k] for q in seqs if k < len(q)]
            lines += len(set(c//16 for c in cols)); ins += 1
    return lines/ins, pad/nz, common_frac/(S1-S0)
def by_col(rows):
    return [pix[pip[r]:pip[r+1]] for r in rows], 0
def common_first(rows):
    offs = [pix[pip[r]:pip[r+1]].astype(np.int64) - r for r in rows]
    common = set(offs[0].tolist())
    for o in offs[1:]: common &= set(o.tolist())
    cs = np.array(sorted(common), dtype=np.int64)
    seqs = []
    for r, o in zip(rows, offs):
        rest = np.setdiff1d(o, cs)
        seqs.append(np.concatenate([cs, rest]) + r)
    return seqs, len(cs)/np.mean([len(o) for o in offs])
S0 = ns//2
for name, f in [("by column", by_col), ("common offsets first", common_first)]:
    print(name, "lines/instr %.2f  slots/nnz %.3f  common frac %.2f" % stats(f, S0, S0+400))
