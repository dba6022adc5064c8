"""Group ncu SASS-level stall samples into regions separated by BAR instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iA, iN = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
tot = sum(float(r[iA] or 0) for r in rows[2:])
reg, regs = [], []
for r in rows[2:]:
    reg.append(r)
    if "BAR" in r[iS] or "WARPSYNC" in r[iS] and False:
        regs.append(reg)
        reg = []
regs.append(reg)
for k, rg in enumerate(regs):
    s = sum(float(r[iA] or 0) for r in rg)
    if s / tot < 0.01:
        continue
    ops = {}
    for r in rg:
        op = r[iS].split()[0] if r[iS].split() else ""
        if op.startswith("@"):
            op = r[iS].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + float(r[iA] or 0)
    st = {}
    for r in rg:
        for i in stall_cols:
            st[h[i]] = st.get(h[i], 0) + float(r[i] or 0)
    top_ops = sorted(ops.items(), key=lambda kv: -kv[1])[:6]
    top_st = sorted(st.items(), key=lambda kv: -kv[1])[:5]
    print(f"region {k}: {len(rg)} instr, {100*s/tot:.1f}% samples; ops " + ", ".join(f"{o}:{100*v/tot:.1f}" for o, v in top_ops))
    print("      stalls " + ", ".join(f"{n.replace('stall_','')}:{100*v/tot:.1f}" for n, v in top_st))
