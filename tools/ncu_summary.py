"""Summarise an ncu --set full report (read here, no GPU) into a JSON list of kernels:
duration, DRAM bytes, achieved DRAM GB/s, tensor / XU / issue utilisation, L2 hit rate.
usage: ncu_summary.py REPORT.ncu-rep OUT.json [kernel-regex]"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = {
    "time_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", None),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", None),
    "xu_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", None),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "registers": ("launch__registers_per_thread", None),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
        "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    rx = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if rx and not rx.search(name):
            continue
        k = {"kernel": re.sub(r"\(.*", "", name).replace("uh::<unnamed>::", "").replace("void ", ""),
             "full_name": name[:200]}
        for key, (m, _) in METRICS.items():
            if m not in h:
                continue
            i = h.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if key == "time_ms":
                v = v * UNIT.get(u, 1.0) * 1e3
            elif key.endswith("_bytes"):
                v = v * UNIT.get(u, 1.0)
            elif key == "sm_clock_ghz":
                v = v * UNIT.get(u, 1.0)
            k[key] = v
        if "time_ms" in k and "dram_read_bytes" in k:
            k["dram_gbs"] = (k["dram_read_bytes"] + k["dram_write_bytes"]) / (k["time_ms"] * 1e-3) / 1e9
        res.append(k)
    json.dump({"report": rep.split("/")[-1], "kernels": res}, open(out, "w"), indent=1)
    for k in res:
        print(f"{k['kernel'][:60]:60s} {k.get('time_ms', 0):8.3f} ms  dram {k.get('dram_gbs', 0):7.0f} GB/s  "
              f"tensor {k.get('tensor_pipe_active_pct', 0):5.1f}%  xu {k.get('xu_pct', 0):5.1f}%")


if __name__ == "__main__":
    main()
