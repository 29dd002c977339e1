"""Summarise an ncu --set full report into profiles/ (key metrics, stall
reasons, top SASS lines).  python tools/ncu_summarize.py REP OUT.txt [json_key]"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main(rep, out, key=None):
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    kname = vals[hdr.index("Kernel Name")]
    m = {}
    lines = [f"# ncu --set full --clock-control none --import-source on: {Path(rep).name}",
             f"kernel: {kname}"]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"{k} = {vals[i]} {units[i]}")
            m[k] = (vals[i], units[i])
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                          "--print-source", "sass"))))
    h = src[1]
    ix = {x: i for i, x in enumerate(h)}
    data = src[2:]

    def f(r, k):
        try:
            return float(r[ix[k]])
        except Exception:
            return 0.0
    tot = sum(f(r, "# Samples") for r in data) or 1.0
    stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    lines.append("warp stall breakdown (% of samples):")
    for s, v in sorted(((s, sum(f(r, s) for r in data)) for s in stalls), key=lambda x: -x[1])[:10]:
        lines.append(f"  {s}: {100 * v / tot:.1f}")
    lines.append("top SASS by samples:")
    for r in sorted(data, key=lambda r: -f(r, "# Samples"))[:15]:
        lines.append(f"  {int(f(r, '# Samples')):>8}  {r[ix['Source']].strip()[:80]}")
    ex = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data)
    al = sum(f(r, "L1 Wavefronts Shared") for r in data)
    lines.append(f"shared wavefronts: {al:.3e} total, {ex:.3e} excessive")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    if key:
        def scale(v, u):
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        summ_path = Path(__file__).resolve().parents[1] / "profiles" / "ncu_summary.json"
        summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
        rd = scale(*m["dram__bytes_read.sum"])
        wr = scale(*m["dram__bytes_write.sum"])
        def pct(k):
            return float(m[k][0]) if k in m else None
        summ[key] = {"report": Path(rep).name, "kernel": kname,
                     "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                     "duration": " ".join(m["gpu__time_duration.sum"]),
                     "fp64_pipe_active_pct":
                         pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                     "dmma_pipe_active_pct": pct(
                         "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
                     "issue_active_pct": pct("sm__throughput.avg.pct_of_peak_sustained_elapsed")}
        summ_path.write_text(json.dumps(summ, indent=1) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
