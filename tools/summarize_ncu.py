"""Text summary of one ncu --set full capture exported as CSV (details / raw / source pages):
tools/summarize_ncu.py DIR TAG  ->  speed-of-light, memory, occupancy, binding units, stall reasons
per SASS line.  Used for the profiles/ summaries of tools/evidence.sh."""
import csv
import os
import sys

d, tag = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(os.path.join(d, f"{tag}_details.csv"))))
h = rows[0]
want = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "SM Active Cycles", "Elapsed Cycles", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Executed Instructions")
kname = None
for r in rows[1:]:
    x = dict(zip(h, r))
    kname = kname or x.get("Kernel Name")
    if x.get("Metric Name") in want:
        print(f"   {x['Metric Name']}: {x['Metric Value']} {x['Metric Unit']}")
rr = list(csv.reader(open(os.path.join(d, f"{tag}_raw.csv"))))
rh, ru, rv = rr[0], rr[1], rr[2]
raw = dict(zip(rh, rv)); unit = dict(zip(rh, ru))
print("# binding units and traffic (raw metrics)")
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed", "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed",
          "lts__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
          "lts__t_requests_srcunit_tex_op_read.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum"):
    if k in raw:
        print(f"   {k} {raw[k]} {unit.get(k, '')}")
print(f"kernel: {kname}")
sys.argv = [sys.argv[0], os.path.join(d, f"{tag}_sass.csv"), "15"]
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_summary  # noqa: E402
sass_summary.main(sys.argv[1], 15)
