"""Summarise ncu reports / launch lists into markdown for profiles/.

usage: python tools/ncu_summary.py launches <launches.csv>
       python tools/ncu_summary.py report <file.ncu-rep> [label]
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
]


def report(path, label):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    print(f"### {label}\n")
    for data in rows[2:]:
        d = dict(zip(h, data))
        u = dict(zip(h, units))
        print(f"kernel: `{d.get('Kernel Name', '?')[:110]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        print()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    per_launch = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ix["ID"]], r[ix["Kernel Name"]])
        try:
            per_launch.setdefault(key, {})[r[ix["Metric Name"]]] = (float(r[ix["Metric Value"]].replace(",", "")),
                                                                    r[ix["Metric Unit"]])
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), m in per_launch.items():
        short = name.split("(")[0].replace("void ", "").split("::")[-1]
        a = agg[short]
        a[0] += 1
        t, unit = m.get("gpu__time_duration.sum", (0.0, "ns"))
        a[1] += t * (1e3 if unit == "us" else 1.0)
        for j, mk in ((2, "dram__bytes_read.sum"), (3, "dram__bytes_write.sum")):
            v, u = m.get(mk, (0.0, "byte"))
            a[j] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    tot = sum(a[1] for a in agg.values())
    print(f"launches in one step: {len(per_launch)}, serialized device time {tot / 1e6:.3f} ms\n")
    print("| kernel | launches | time (us) | share | DRAM read (MB) | DRAM write (MB) |\n|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {a[0]} | {a[1] / 1e3:.1f} | {a[1] / tot * 100:.1f}% | {a[2] / 1e6:.1f} | {a[3] / 1e6:.1f} |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[2])
