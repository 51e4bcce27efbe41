"""Summarise one-kernel ncu captures (--set full) into the numbers profiles/ and bench.py use.

    python tools/ncu_summarize.py gpurun_out/r02_sweep2m.ncu-rep [more.ncu-rep ...]

Prints one JSON object per report: duration, DRAM bytes, L2/L1 hit rates, SM / issue / warp
occupancy, fp64-pipe and shared-memory activity, instruction counts, registers, smem.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "dram__bytes.sum.per_second": "dram_bytes_per_s",
    "lts__t_sectors.sum": "l2_sectors",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__inst_executed_pipe_fp64.sum": "fp64_warp_inst",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__inst_executed.sum": "sm_warp_inst",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed": "smem_pipe_pct",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic_bytes",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "smsp__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "smsp_fp64_pipe_pct",
}


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {"report": path}
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        res["kernel"] = rec.get("Kernel Name", "")[:120]
        for k, name in WANT.items():
            if k in rec and rec[k] not in ("", "n/a"):
                v = rec[k].replace(",", "")
                try:
                    val = float(v)
                except ValueError:
                    continue
                unit = (units[hdr.index(k)] if k in hdr else "").split("/")[0]
                val *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1.0,
                        "nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
                        "second": 1e9, "s": 1e9, "Tbyte": 1e12}.get(unit, 1.0)
                res[name] = val
        break
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps(summarize(p)))
