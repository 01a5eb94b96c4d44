"""Summarise an ncu --set full report of one of our kernels into a text file
for profiles/: speed-of-light, issue/pipe utilisation, shared-memory
wavefronts, DRAM traffic per launch, and the per-role (producer / consumer
warps) instruction mix and stall breakdown.
usage: python tools/ncu_summary.py report.ncu-rep [out.txt] [--stats KEY pixels pairs]
  --stats: also record the launch's DRAM bytes and MUFU (XU-pipe) lane-ops
  per launch under KEY in profiles/kernel_stats.json (read by bench.py for
  roofline.traffic and roofline.sfu); pixels x pairs = the launch's
  pixel-pairs, for the per-pixel-pair MUFU count."""
import collections
import csv
import io
import re
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    lines = []
    raw = ncu_csv(rep, "--page", "raw")
    h, units, vals = raw[0], raw[1], raw[2]
    d = {h[i]: (vals[i], units[i]) for i in range(len(h))}
    lines.append(f"report: {rep}")
    lines.append(f"kernel: {d.get('Kernel Name', ('?', ''))[0]}")
    keys = [
        ("gpu__time_duration.sum", "duration"),
        ("sm__cycles_elapsed.avg.per_second", "SM clock"),
        ("launch__grid_size", "grid"),
        ("launch__block_size", "block"),
        ("launch__registers_per_thread", "registers/thread"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
        ("smsp__warps_active.avg.per_cycle_active", "active warps/scheduler"),
        ("smsp__inst_executed.sum", "warp instructions"),
    ]
    for k, name in keys:
        if k in d:
            lines.append(f"  {name:28s} {d[k][0]} {d[k][1]}")
    # per-role breakdown from the SASS source page
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    sh = src[1]
    si, ei = sh.index("Source"), sh.index("Instructions Executed")
    stalls = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    ops = {"P": collections.Counter(), "C": collections.Counter()}
    st = {"P": collections.Counter(), "C": collections.Counter()}
    has_alloc = any("TRY_ALLOC" in r[si] for r in src[2:])
    region = "P"
    for r in src[2:]:
        s = r[si].strip()
        if region == "P" and (("TRY_ALLOC" in s) if has_alloc else s.startswith("EXIT")):
            region = "C"
        op = re.sub(r"^@!?U?P[0-9T]+\s+", "", s).split(" ")[0].split(".")[0]
        ops[region][op] += int(r[ei] or 0)
        for c in stalls:
            st[region][c] += int(r[sh.index(c)] or 0)
    for k, name in (("P", "producer warps"), ("C", "consumer warps")):
        tot = sum(ops[k].values()) or 1
        lines.append(f"{name}: {tot} warp-instr; ops: " +
                     ", ".join(f"{o} {v / tot:.1%}" for o, v in ops[k].most_common(10)))
        ts = sum(st[k].values()) or 1
        lines.append(f"  stalls ({ts} samples): " +
                     ", ".join(f"{c[6:]} {v / ts:.1%}" for c, v in st[k].most_common(8)))
    text = "\n".join(lines) + "\n"
    args = sys.argv[2:]
    if "--stats" in args:
        i = args.index("--stats")
        key, pixels, pairs = args[i + 1], float(args[i + 2]), float(args[i + 3])
        args = args[:i] + args[i + 4:]
        tu = d["gpu__time_duration.sum"][1]
        cycles = float(d["gpu__time_duration.sum"][0]) * {"ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6,
                                                          "ns": 1e-9, "nsecond": 1e-9}.get(tu, 1.0)   # seconds
        clk = float(d["sm__cycles_elapsed.avg.per_second"][0]) * (1e9 if "Ghz" in d["sm__cycles_elapsed.avg.per_second"][1]
                                                                  else 1e6)
        sms = float(d["device__attribute_multiprocessor_count"][0]) if "device__attribute_multiprocessor_count" in d else 148
        xu = float(d["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"][0]) / 100.0 * 16 * sms * cycles * clk

        def mb(k):
            v, u = d[k]
            return float(v) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
        import json
        import os
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "kernel_stats.json")
        stats = json.load(open(path)) if os.path.exists(path) else {}
        stats[key] = {"dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                      "mufu_lane_ops_per_launch": xu, "mufu_per_pixel_pair": xu / (pixels * pairs),
                      "kernel": d.get("Kernel Name", ("?", ""))[0],
                      "source": f"ncu --set full capture {os.path.basename(rep)} "
                                f"(XU pipe {float(d['sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'][0]):.1f} % "
                                f"of 16 lanes/clk/SM over {cycles * 1e3:.3f} ms)"}
        json.dump(stats, open(path, "w"), indent=1)
    if args:
        open(args[0], "w").write(text)
    print(text, end="")


if __name__ == "__main__":
    main()
