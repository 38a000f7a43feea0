"""Summarise an .ncu-rep: key throughput metrics and top stall reasons per
kernel launch.   python tools/ncu_summary.py gpurun_out/prof.ncu-rep
With --json N POINTS SOURCE: print profiles/ncu_summary.json (the DRAM
traffic per launch bench.py reports as roofline.traffic) for the first
launch in the report."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        print("==", r[hdr.index("Kernel Name")][:90])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k:70s} {r[i]:>14s} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("   stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(st, reverse=True)[:8]))


def to_json(path, N, points, source):
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, r = rows[0], rows[1], rows[2]

    def val(k):
        v = float(r[hdr.index(k)].replace(",", ""))
        u = units[hdr.index(k)]
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    dur = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
    print(json.dumps({
        "N": N, "world": 1, "kernel": r[hdr.index("Kernel Name")][:120],
        "dram_bytes_per_launch": rd + wr, "dram_read_bytes_per_launch": rd,
        "dram_write_bytes_per_launch": wr, "ncu_duration_ms": [dur],
        "points_per_launch": points, "dram_bytes_per_update": (rd + wr) / (2 * points),
        "source": source}, indent=1))


if __name__ == "__main__":
    if "--json" in sys.argv:
        i = sys.argv.index("--json")
        to_json(sys.argv[1], int(sys.argv[i + 1]), int(sys.argv[i + 2]), sys.argv[i + 3])
    else:
        main(sys.argv[1])
