"""Summarise an ncu report: key raw metrics + stall reasons + top SASS lines."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, val = rows[0], rows[1], rows[-1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for w in want:
    for i, h in enumerate(hdr):
        if h == w:
            print(f"{w:65s} {val[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0.0 for h in st}
for r in data:
    for h in st:
        try: tot[h] += float(r[idx[h]] or 0)
        except ValueError: pass
S = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{h[6:]} {v/S*100:.0f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
if len(sys.argv) > 2:
    top = sorted(data, key=lambda r: -float(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2])]
    for r in top:
        print(r[idx["Warp Stall Sampling (All Samples)"]], r[idx["Address"]], r[idx["Source"]][:80])
