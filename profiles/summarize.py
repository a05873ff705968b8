#!/usr/bin/env python3
"""Summarise ncu outputs brought back in gpurun_out/ into the committed
profiles/ files (run in the build container; ncu -i works without a GPU).

  python profiles/summarize.py launches <launch-list.csv> <out.txt>
      one steady-state substep of the bench command (kernel, device time, share)
  python profiles/summarize.py full <report.ncu-rep> <out.txt> [--traffic profiles/traffic.json]
      key metrics per profiled kernel; with --traffic, the measured DRAM bytes
      per launch of each kernel are recorded for bench.py's roofline.traffic
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_instr"),
    ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "l2_atomic_%"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "l2_red_sectors"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_bank_conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem_st_bank_conflicts"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "smem_ld_instr"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local_ld_instr"),
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    seq = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        seq.append((r[ki].split("(")[0].replace("void ", ""), v))
    starts = [i for i, (n, _) in enumerate(seq) if "status_reset" in n] + [len(seq)]
    # steady-state substeps of the device-timed loop: windows between status
    # resets holding a P2G launch and no upload / initial-stress / full-sort
    # kernels; the median-length one is reported
    wins = []
    for a, b in zip(starts[:-1], starts[1:]):
        names = [n for n, _ in seq[a:b]]
        if not any("p2g" in n for n in names):
            continue
        if any(("aos" in n) or ("stress_kernel" in n) or ("iota" in n) for n in names):
            continue
        wins.append((sum(v for _, v in seq[a:b]), a, b))
    wins.sort()
    _, s, e = wins[len(wins) // 2]
    step = seq[s:e]
    tot = sum(v for _, v in step)
    with open(out, "w") as f:
        f.write(f"# one steady-state substep of the bench command, ncu gpu__time_duration.sum\n")
        f.write(f"# (cold-cache, serialised launches: compare SHARES, not absolutes)\n")
        f.write(f"# source: {path}\n")
        for n, v in step:
            f.write(f"{n:48s} {v / 1e3:10.1f} us  {v / tot * 100:5.1f} %\n")
        f.write(f"{'substep total':48s} {tot / 1e3:10.1f} us\n")
        agg = collections.OrderedDict()
        for n, v in seq:
            agg.setdefault(n, []).append(v)
        f.write("\n# all launches of the run, by kernel\n")
        for n, vs in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{n:48s} n={len(vs):4d} avg={sum(vs) / len(vs) / 1e3:10.1f} us\n")
    print(open(out).read())


def full(path, out, traffic=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    by_kernel = collections.OrderedDict()
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        by_kernel.setdefault(name, []).append(r)
    lines = [f"# ncu --set full summary; source: {path}"]
    tr = {}
    for name, rs in by_kernel.items():
        lines.append(f"\n== {name}  ({len(rs)} launch(es) profiled)")
        for m, label in METRICS:
            if m not in h:
                continue
            i = h.index(m)
            vals = []
            for r in rs:
                try:
                    vals.append(float(r[i].replace(",", "")))
                except ValueError:
                    pass
            if vals:
                lines.append(f"  {label:26s} {sum(vals) / len(vals):14.4f} {units[i]}")
        short = name.split("::")[-1].split("<")[0]
        def avg(m):
            i = h.index(m)
            return sum(float(r[i].replace(",", "")) for r in rs) / len(rs)

        if "dram__bytes_read.sum" in h:
            # each metric in its own unit (ncu picks Mbyte/Gbyte per value)
            to_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = avg("dram__bytes_read.sum") * to_b.get(units[h.index("dram__bytes_read.sum")], 1)
            wr = avg("dram__bytes_write.sum") * to_b.get(units[h.index("dram__bytes_write.sum")], 1)
            tr[short.replace("_tile", "")] = rd + wr
        # floating-point operation counts (thread-level SASS ops; FMA = 2 flops):
        # per-cycle rates summed over SMSPs x elapsed SMSP cycles
        cyc = "smsp__cycles_elapsed.avg"
        if cyc in h:
            for prec, ops in (("fp64", ("dadd", "dmul", "dfma")), ("fp32", ("fadd", "fmul", "ffma"))):
                ms = [f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed" for o in ops]
                if not all(m in h for m in ms):
                    continue
                cnt = [avg(m) * avg(cyc) for m in ms]
                fl = cnt[0] + cnt[1] + 2 * cnt[2]
                if fl > 0:
                    lines.append(f"  {prec + '_ops add/mul/fma':26s} {cnt[0]:.4e} / {cnt[1]:.4e} / {cnt[2]:.4e}")
                    tu = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}
                    secs = avg("gpu__time_duration.sum") * tu.get(units[h.index("gpu__time_duration.sum")], 1)
                    lines.append(f"  {prec + '_flop':26s} {fl:14.4e} ({fl / secs / 1e12:.2f} TFLOP/s)")
    # stall reasons of the longest kernel
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic:
        try:  # keep the file's other keys (e.g. fp64_flop_per_launch)
            merged = json.load(open(traffic))
        except (OSError, ValueError):
            merged = {}
        merged.update(tr)
        json.dump(merged, open(traffic, "w"), indent=1)
        print("traffic:", tr)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        t = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
        full(sys.argv[2], sys.argv[3], t)
