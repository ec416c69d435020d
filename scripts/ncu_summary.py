"""Summarise an ncu report (raw page) into a small JSON + text (for profiles/)."""
import csv, io, json, subprocess, sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_bytes.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    rep, out = sys.argv[1], sys.argv[2]
    res = summarise(rep)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for d in res:
        print(json.dumps(d, indent=1))
