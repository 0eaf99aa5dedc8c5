"""Summarise ncu reports / launch lists into markdown for profiles/ (run locally on the
.ncu-rep / csv files brought back from gpurun)."""
import collections
import csv
import subprocess
import sys

SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "msecond": 1e3,
         "usecond": 1.0, "nsecond": 1e-3}


def raw_rows(rep):
    """rep: an .ncu-rep, or the `ncu -i rep --page raw --csv` export of one (.csv)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [{h: (u, v) for h, u, v in zip(hdr, units, r)} for r in rows[2:]]


def val(d, key, to=None):
    if key not in d:
        return float("nan")
    u, v = d[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return float("nan")
    if to and u in SCALE:
        x *= SCALE[u]
    return x


def full_table(rep, title, note):
    rows = raw_rows(rep)
    lines = [f"# {title}", "", note, "",
             "| kernel | grid x block | duration (us) | DRAM rd (MB) | DRAM wr (MB) | DRAM GB/s | tensor-pipe smem cycles active (%) | HMMA/UTC inst (% of peak) | SM throughput (%) | issue slots busy (%) | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in rows:
        name = d["Kernel Name"][1].split("(")[0].replace("void ", "").replace("ng::<unnamed>::", "").replace("ng::", "")
        t = val(d, "gpu__time_duration.sum", "us")
        rd = val(d, "dram__bytes_read.sum", "MB")
        wr = val(d, "dram__bytes_write.sum", "MB")
        lines.append(
            f"| `{name}` | {d['Grid Size'][1]} x {d['Block Size'][1]} | {t:.1f} | {rd:.2f} | {wr:.2f} | "
            f"{(rd + wr) / t * 1e3:.0f} | {val(d, 'sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{val(d, 'sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active'):.2f} | "
            f"{val(d, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{val(d, 'sm__instruction_throughput.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{d.get('launch__registers_per_thread', ('', ''))[1]} |")
    return "\n".join(lines) + "\n"


def launch_table(csv_path, steps, title, marker="input_kernel"):
    rows = list(csv.reader(open(csv_path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    idx = [i for i, d in enumerate(data) if d["Kernel Name"].startswith(marker)]
    sub = data[idx[-steps - 1]:idx[-1]]   # `steps` whole steps, ending at the last step's start (later
                                          # launches -- bench.py's standalone preconditioner run -- excluded)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in sub:
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("ng::<unnamed>::", "").replace("ng::", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {title}", "",
             f"`ncu --metrics gpu__time_duration.sum --clock-control none` launch list, last {steps} steps of "
             "`bench.py --steps 24 --warmup 10` (kernels serialised and cold under ncu: compare SHARES; side-stream "
             "kernels overlap the main stream in a real run).", "",
             "| kernel | launches/step | us/launch | us/step | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0] / steps:.2f} | {v[1] / v[0] / 1e3:.1f} | {v[1] / steps / 1e3:.1f} | {100 * v[1] / tot:.1f}% |")
    lines.append(f"| **total (serialised)** | {sum(v[0] for v in agg.values()) / steps:.1f} | | {tot / steps / 1e3:.1f} | 100% |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    kind = sys.argv[1]
    if kind == "full":
        print(full_table(sys.argv[2], sys.argv[3], sys.argv[4]))
    else:
        print(launch_table(sys.argv[2], int(sys.argv[3]), sys.argv[4]))
