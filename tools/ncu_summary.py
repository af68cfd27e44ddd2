"""Summarise `ncu --set full` reports (raw page) into profiles/<round>_ncu_summary.json.

usage: python tools/ncu_summary.py out.json report1.ncu-rep [report2.ncu-rep ...]
Keeps, per profiled launch: duration, DRAM bytes read/written, DRAM and tensor
pipe utilisation, issue activity, occupancy, registers and grid size.  The
first decode_tcd_kernel / decode_kernel launch's DRAM bytes become decode_traffic_bytes_per_launch
(bench.py's roofline "traffic")."""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for v in r[2:]:
        yield {h: (x, u) for h, x, u in zip(hdr, v, units)}


def main():
    dst, reps = sys.argv[1], sys.argv[2:]
    kernels, traffic = [], None
    for rep in reps:
        for d in rows(rep):
            k = {"kernel": d["Kernel Name"][0][:90], "report": rep.split("/")[-1]}
            for m in KEEP:
                if m in d:
                    k[m] = [d[m][0], d[m][1]]
            kernels.append(k)
            if traffic is None and ("decode_tcd_kernel" in k["kernel"] or "decode_kernel" in k["kernel"]):
                b = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    x, u = d[m]
                    b += float(x.replace(",", "")) * UNIT.get(u, 1)
                traffic = b
    json.dump({"source": "ncu --set full --clock-control none (tools/ncu_summary.py)", "kernels": kernels,
               "decode_traffic_bytes_per_launch": traffic}, open(dst, "w"), indent=1)
    print(f"{len(kernels)} launches -> {dst}; decode traffic/launch {traffic}")


if __name__ == "__main__":
    main()
