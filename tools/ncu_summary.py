"""Summarise ncu reports: per kernel launch, the metrics the roofline
discussion uses (duration, DRAM bytes, pipe utilisation, smem/L2 traffic,
registers, occupancy).  python tools/ncu_summary.py rep1.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_tc_read_%"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed", "xbar2l1_fill_%"),
    ("lts__t_bytes.sum.pct_of_peak_sustained_elapsed", "l2_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__grid_size", "grid"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for v in r[2:]:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        yield d, u


def main():
    print("| report | kernel | " + " | ".join(n for _, n in KEYS) + " |")
    print("|" + "---|" * (len(KEYS) + 2))
    for rep in sys.argv[1:]:
        for d, u in rows(rep):
            name = d.get("Kernel Name", "?")[:70]
            vals = []
            for k, n in KEYS:
                v = d.get(k, "") or next((d[h] for h in d if h.endswith(k) and d[h]), "")
                vals.append(f"{v} {u.get(k, '')}".strip() if v else "-")
            print(f"| {rep.split('/')[-1]} | `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
