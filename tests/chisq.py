"""Per-(prev, cur) transition chi-square against the exact dynamic
probabilities (oracle.transition_probs = the reference's oracle_enumerate,
samplers.hpp:272-288).

Walkers start at s; their step-2 moves from cur = path[1] with prev = s are
samples of the (s, cur) transition.  Groups with enough samples are tested
cell by cell (cells with expected count < 5 pooled); returns the per-group
p-values and the pooled p-value (sum of statistics, sum of degrees of
freedom)."""
import numpy as np
from scipy.stats import chi2


def transition_pvalues(orc, og, model, paths, starts, min_n=400):
    row = og.arrays()["row"]
    col = og.arrays()["col"]
    ps, stat, dof = [], 0.0, 0
    for s in np.unique(starts):
        sel = (starts == s) & (paths[:, 2] != 0xFFFFFFFF)
        cur = paths[sel, 1]
        nxt = paths[sel, 2]
        for c in np.unique(cur):
            m = cur == c
            n = int(m.sum())
            if n < min_n:
                continue
            probs = orc.transition_probs(og, model, int(c), int(s), 1)
            if probs is None:
                continue
            tgt = col[row[c]:row[c + 1]]
            # probability per distinct target (multigraph rows may repeat one)
            uniq, inv = np.unique(tgt, return_inverse=True)
            p = np.bincount(inv, weights=probs, minlength=len(uniq))
            obs = np.bincount(np.searchsorted(uniq, nxt[m]), minlength=len(uniq)).astype(float)
            assert np.all(np.isin(nxt[m], uniq)), "a step left the row"
            exp = p * n
            big = exp >= 5
            o = np.append(obs[big], obs[~big].sum())
            e = np.append(exp[big], exp[~big].sum())
            keep = e > 0
            o, e = o[keep], e[keep]
            if len(o) < 2:
                continue
            x = float(((o - e) ** 2 / e).sum())
            k = len(o) - 1
            ps.append(float(chi2.sf(x, k)))
            stat += x
            dof += k
    pooled = float(chi2.sf(stat, dof)) if dof else 1.0
    return ps, pooled
