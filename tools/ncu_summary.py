"""Developer tool: condensed summary of one kernel in an .ncu-rep (speed of
light, memory, occupancy, stall reasons, L2/DRAM traffic by op)."""
import csv
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread",
        "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler", "Memory Throughput",
        "Mem Busy", "Max Bandwidth", "Compute (SM) Throughput", "Grid Size", "Block Size")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
       "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
       "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
       "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "smsp__inst_executed.sum", "sm__cycles_elapsed.avg")


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    name = None
    for r in rows[1:]:
        if len(r) > 14:
            name = name or r[4]
            if r[12] in KEYS:
                print(f"  {r[12]:34s} {r[14]:>14s} {r[13]}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
    units = dict(zip(rows[0], rows[1])) if len(rows) > 2 else {}
    st = []
    for k, x in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(x.replace(",", "")), k.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    print("  stalls (cycles per issued instruction):",
          ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    for k in RAW:
        if k in d:
            print(f"  {k:58s} {d[k]:>18s} {units.get(k, '')}")
    print("  kernel:", (name or "?")[:100])


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(rep)
        main(rep)
