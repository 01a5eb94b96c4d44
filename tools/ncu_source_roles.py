"""Summarise an `ncu --page source --csv --print-source sass` export of the v7
kernel by role: instructions are assigned to the consumer pair loop, the
producer pair loop (unrolled UNR deep), the mbarrier spin loop or the rest
(prologues, segment inits, epilogues) by their execution counts, and the warp
stall samples of each group are broken down by reason.  Usage:
    python tools/ncu_source_roles.py gpurun_out/src_sass.csv [steps_per_warp]"""
import collections
import csv
import sys

KEYS = ["long_sb", "wait", "short_sb", "mio", "math", "selected", "not_selected", "dispatch",
        "branch_resolving", "no_inst", "lg", "barrier", "sleep", "misc"]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (KeyError, ValueError):
            return 0.0

    execs = sorted(f(r, "Instructions Executed") for r in data)
    # the consumer pair loop is not unrolled: its instructions share the
    # count carrying the most executed warp-instructions
    classes = collections.Counter(execs)
    cons_n = max(classes, key=lambda e: e * classes[e])
    groups = collections.defaultdict(collections.Counter)
    top = collections.defaultdict(list)

    def role(e):
        if abs(e - cons_n) <= 0.03 * cons_n:
            return "consumer pair loop"
        if e > 1.5 * cons_n:
            return "mbarrier spin"
        if 0.08 * cons_n < e < 0.2 * cons_n:
            return "producer pair loop"
        return "other (prologues, inits, epilogues)"

    for r in data:
        e = f(r, "Instructions Executed")
        g = role(e)
        c = groups[g]
        c["samples"] += f(r, "Warp Stall Sampling (All Samples)")
        c["instr"] += 1
        c["exec"] += e
        for k in KEYS:
            c[k] += f(r, "stall_" + k)
        op = r[ix["Source"]].split()
        op = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")
        c["op:" + op.split(".")[0]] += e
        top[g].append((f(r, "Warp Stall Sampling (All Samples)"), r[ix["Source"]].strip()[:70]))
    total = sum(c["samples"] for c in groups.values())
    print(f"source: {path}")
    print(f"kernel: {rows[0][1] if len(rows[0]) > 1 else '?'}")
    print(f"warp-stall samples: {int(total)}; consumer pair-loop instruction executed {int(cons_n)} times")
    for g, c in sorted(groups.items(), key=lambda kv: -kv[1]["samples"]):
        print(f"\n== {g}: {100 * c['samples'] / total:.1f}% of samples, {int(c['instr'])} SASS instructions, "
              f"{c['exec']:.3g} warp-instr executed")
        print("   stalls: " + ", ".join(f"{k} {100 * c[k] / c['samples']:.1f}%" for k in KEYS
                                       if c[k] > 0.01 * c["samples"]))
        ops = sorted(((v, k[3:]) for k, v in c.items() if k.startswith("op:")), reverse=True)[:10]
        print("   mix:    " + ", ".join(f"{o} {100 * v / c['exec']:.1f}%" for v, o in ops))
        for s, src in sorted(top[g], reverse=True)[:5]:
            print(f"   top: {int(s):6d}  {src}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/src_sass.csv")
