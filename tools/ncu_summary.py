"""Summarise ncu reports (offline) into profiles/.

    python tools/ncu_summary.py OUT_PREFIX REPORT.ncu-rep [REPORT2 ...]

Writes OUT_PREFIX.md (human-readable table) and OUT_PREFIX.json (per-kernel
metrics: duration, DRAM bytes, pipe utilisation, issue, occupancy, stall
breakdown).  bench.py reads the dram bytes from profiles/ncu_traffic.json.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "sm_mhz": "sm__cycles_elapsed.avg.per_second",
    "regs": "launch__registers_per_thread",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    # ncu 2025 exposes the fmaheavy pipe only as ..._elapsed (the _active form is absent)
    "fmaheavy_pipe_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "fmaheavy_inst_pct": "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_elapsed",
    "elapsed_cycles": "sm__cycles_elapsed.avg",
    "inst_executed": "smsp__inst_executed.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "dram_pct_peak": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for v in r[2:]:
        yield dict(zip(hdr, v)), dict(zip(hdr, units))


def fnum(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def scale(val, unit, want):
    if val is None:
        return None
    f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    if want == "MB" and unit in f:
        return val * f[unit]
    if want == "us":
        return {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0) * val
    if want == "MHz":
        return {"hz": 1e-6, "Khz": 1e-3, "Mhz": 1.0, "Ghz": 1e3, "cycle/second": 1e-6,
                "cycle/nsecond": 1e3, "cycle/usecond": 1.0}.get(unit, 1.0) * val
    return val


def fmt(v):
    return "-" if v is None else f"{v:.0f}"


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    allk = []
    for rep in reps:
        for d, u in rows(rep):
            k = {"report": rep.split("/")[-1], "kernel": d.get("Kernel Name", "")[:90], "id": d.get("ID")}
            for name, key in KEYS.items():
                v = fnum(d.get(key))
                if name.endswith("_MB"):
                    v = scale(v, u.get(key, ""), "MB")
                elif name == "duration_us":
                    v = scale(v, u.get(key, ""), "us")
                elif name == "sm_mhz":
                    v = scale(v, u.get(key, ""), "MHz")
                k[name] = v
            # every fmaheavy / fma / alu pipe counter the report holds (names vary by ncu version)
            k["pipes"] = {key: fnum(val) for key, val in d.items()
                          if ("pipe_fmaheavy" in key or "pipe_alu" in key or "pipe_fma_" in key)
                          and fnum(val) is not None}
            stalls = {}
            for key, val in d.items():
                if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                    nm = key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                    fv = fnum(val)
                    if fv and fv >= 0.05:
                        stalls[nm] = round(fv, 3)
            k["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
            allk.append(k)
    json.dump(allk, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write("| kernel | us | DRAM R/W MB | regs | warps act % | issue % | fma pipe % | fmaheavy % | alu pipe % | top stalls (cycles/issue) |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for k in allk:
            st = ", ".join(f"{a} {b}" for a, b in list(k["stalls_per_issue"].items())[:5])
            f.write(f"| {k['kernel'][:48]} | {k['duration_us']:.1f} | {k['dram_read_MB']:.1f}/{k['dram_write_MB']:.1f} | "
                    f"{k['regs']:.0f} | {k['warps_active_pct']:.0f} | {k['issue_active_pct']:.0f} | "
                    f"{k['fma_pipe_pct']:.0f} | {fmt(k.get('fmaheavy_pipe_pct'))} | {k['alu_pipe_pct']:.0f} | {st} |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
