"""Summarise an ncu --set full report: one row per kernel launch with duration, DRAM bytes,
achieved DRAM GB/s, SM / L1 / L2 / issue utilisation and occupancy (reads `ncu -i --page raw --csv`)."""
import csv
import io
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_cyc_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "launch__registers_per_thread": "regs",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wf",
    "sm__cycles_elapsed.avg": "cycles",
}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    ki = hdr.index("Kernel Name")
    print(f"{'kernel':34s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>7s} " + " ".join(f"{METRICS[m]:>9s}" for m in idx if m not in ('gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum')))
    units = rows[1]
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in rows[2:]:
        def val(m):
            try:
                return float(r[idx[m]].replace(",", "")) * scale.get(units[idx[m]], 1.0)
            except Exception:
                return float("nan")
        dur = val("gpu__time_duration.sum")      # ns
        unit_scale = 1e-3  # ns -> us
        dram = (val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
        print(f"{r[ki][:34]:34s} {dur * unit_scale:8.1f} {dram / 1e6:9.1f} {dram / (dur * 1e-9) / 1e9:7.0f} " +
              " ".join(f"{val(m):9.1f}" for m in idx if m not in ('gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum')))


if __name__ == "__main__":
    main(sys.argv[1])
