"""Summarise ncu --set full reports: one row per captured launch with the
metrics the profiles/ READMEs quote (duration, clock, tensor-pipe activity,
DRAM bytes and bandwidth, L2 hit rate, registers, grid)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "gpc__cycles_elapsed.max.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for vals in r[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        yield d.get("Kernel Name", "?"), {k: (d.get(k, ""), u.get(k, "")) for k in KEYS}


if __name__ == "__main__":
    w = csv.writer(sys.stdout)
    w.writerow(["report", "kernel"] + KEYS)
    for rep in sys.argv[1:]:
        for name, m in rows(rep):
            w.writerow([rep.split("/")[-1], name[:60]] + [f"{v} {u}".strip() for v, u in m.values()])
