"""Prints the bit geometry of plan steps (host only, no GPU): for the big operand X
and the output O of a bond-2 step, which bits are M (X bit -> O bit), K (X bit,
contracted) and N (O bit from the small operand). Bit i = axis rank-1-i
(canonical row-major layout, runtime.hpp:341-346)."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2005_06787_b200.runtime import load_desc

path, steps = sys.argv[1], [int(x) for x in sys.argv[2:]]
d = load_desc(path).contents
for si in steps:
    s = d.steps[si]
    lr, rr, orank = s.lrank, s.rrank, s.orank
    lperm = [s.lperm[i] for i in range(lr)]
    rperm = [s.rperm[i] for i in range(rr)]
    operm = [s.operm[i] for i in range(orank)]
    nd, nm, nk, nn = s.nd, s.nm, s.nk, s.nn
    # produced axis p -> source: D/M from lhs axis lperm[p]; N from rhs axis rperm[nd+nk+(p-nd-nm)]
    lbits = lambda ax: lr - 1 - ax
    rbits = lambda ax: rr - 1 - ax
    obits = lambda ax: orank - 1 - ax
    big_is_l = s.M * s.K >= s.K * s.N
    roles = []
    for i in range(orank):
        p = operm[i]
        if p < nd:
            roles.append(("D", obits(i), lbits(lperm[p]), rbits(rperm[p])))
        elif p < nd + nm:
            roles.append(("M", obits(i), lbits(lperm[p]), None))
        else:
            q = p - nd - nm
            roles.append(("N", obits(i), None, rbits(rperm[nd + nk + q])))
    kroles = [("K", None, lbits(lperm[nd + nm + q]), rbits(rperm[nd + q])) for q in range(nk)]
    print(f"step {si} D={s.D} M={s.M} N={s.N} K={s.K} lrank={lr} rrank={rr} orank={orank} "
          f"branch={s.is_branch} big={'lhs' if big_is_l else 'rhs'}")
    allr = sorted(roles, key=lambda r: r[1])
    print("  O bits low->high:", " ".join(f"{r[0]}{'' if r[2] is None else 'x'+str(r[2])}{'' if r[3] is None else 'w'+str(r[3])}" for r in allr[:16]))
    print("  K:", " ".join(f"l{r[2]}/r{r[3]}" for r in kroles))
