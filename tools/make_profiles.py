"""Turn raw ncu outputs (gpurun_out/) into the committed summaries under profiles/.

  python tools/make_profiles.py launches gpurun_out/launches.csv r01 "<command>"
      ncu --metrics gpu__time_duration.sum --clock-control none --csv log of a
      bench run -> profiles/<tag>_launches_summary.txt (last RHS: per-kernel time
      and share; cold-cache, serialised per-launch times — compare shares)
  python tools/make_profiles.py full gpurun_out/rhs_full.ncu-rep r01 "<command>"
      ncu --set full capture of one RHS -> profiles/<tag>_rhs_full_ncu.txt and
      profiles/<tag>_roofline_traffic.json (DRAM bytes per launch, keyed "passA d=5")

Kernels are attributed to orders from their grid: pass A launches npairs*N2
CTAs, pass B ceil(K_rows/8) with K_rows ~ d*N1/2; pass C follows its order's
pass B, qcoef its order's pass A (in pass-A issue order).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N1, N2 = 4096, 256  # C5 geometry at N = 2^20
C5_PAIRS = {300: 5, 48: 4, 9: 3, 2: 2}


def short(name):
    name = re.sub(r"\(.*\)$", "", name.replace("<unnamed>::", "").replace("(anonymous namespace)::", ""))
    return name.replace("void ", "").strip()


def grid_count(g):
    nums = [int(x) for x in re.findall(r"\d+", g)]
    out = 1
    for x in nums:
        out *= x
    return out


def label(rows):
    """[(kernel, grid, value...)] in issue order -> labels 'passA d=5' etc.
    Pass A: the grid gives the order for the one-CTA-per-item kernels
    (npairs x N2 CTAs); the persistent TMA-fed pass A launches a fixed grid,
    so its launches are labelled by issue order (cheapest order first, the
    costliest last: run_orders).  qcoef launches belong to the oldest pass A
    whose qcoef has not been seen yet; pass C follows its own order's pass B."""
    out, cur, pending = [], None, []
    a_order = sorted(C5_PAIRS.values())
    na = 0
    for name, grid in rows:
        k = short(name)
        if k.startswith("passA"):
            cur = C5_PAIRS.get(grid // N2) if k.startswith("passA_big") or k.startswith("passA_kernel") else None
            if cur is None:
                cur = a_order[min(na, len(a_order) - 1)]
            na += 1
            pending.append(cur)
            out.append(f"passA d={cur}")
        elif k.startswith("passB"):
            cur = round(grid / (N1 // 16))
            out.append(f"passB d={cur}")
        elif k.startswith("passC"):
            out.append(f"passC d={cur}")
        elif k.startswith("qcoef"):
            out.append(f"qcoef d={pending.pop(0) if pending else None}")
        else:
            out.append(k)
    return out


def launches(path, tag, command):
    text = open(path).read()
    body = text[text.index('"ID"'):]
    rows = [r for r in csv.DictReader(io.StringIO(body)) if r["Metric Name"] == "gpu__time_duration.sum"]
    names = [short(r["Kernel Name"]) for r in rows]
    # last complete device RHS (rhs_device): permute -> pass A ... -> combine_natural
    ends = [i for i, n in enumerate(names) if n.startswith("combine_natural")]
    starts = [i for i, n in enumerate(names) if n.startswith("permute") and names[i + 1].startswith("passA")]
    segs = []  # complete C5 RHS evaluations (the order-5 pass A has 300 pairs x N2 CTAs)
    for a in starts:
        b = next((e for e in ends if e > a), None)
        if b is not None and sum(names[i].startswith("passA") for i in range(a, b)) == len(C5_PAIRS):
            segs.append((a, b))
    a, b = segs[-1]
    seg = rows[a: b + 1]
    labs = label([(r["Kernel Name"], grid_count(r["Grid Size"])) for r in seg])
    ns = [float(r["Metric Value"]) for r in seg]
    tot = sum(ns)
    agg = {}
    for lab, v in zip(labs, ns):
        agg[lab] = agg.get(lab, 0.0) + v
    lines = [f"ncu --metrics gpu__time_duration.sum --clock-control none; command: {command}",
             "per-launch device time of the last RHS, cold-cache and serialised under ncu: compare SHARES, not absolutes",
             "(in the timed bench the cheaper orders' pass B/C run on a least-priority stream that fills the SMs the costliest order leaves idle)", ""]
    for lab, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"{lab:28s} {v / 1e3:10.1f} us   {v / tot * 100:5.1f}%")
    lines += ["", f"{'total':28s} {tot / 1e3:10.1f} us over {len(seg)} launches per RHS", "",
              "launches in issue order:"]
    for r, lab, v in zip(seg, labs, ns):
        lines.append(f"  {lab:24s} {short(r['Kernel Name']):40s} grid {r['Grid Size']:>16s} {v / 1e3:10.1f} us")
    out = os.path.join(ROOT, "profiles", f"{tag}_launches_summary.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
]
TO_BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def full(rep, tag, command):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    labs = label([(r[ix["Kernel Name"]], int(float(r[ix["launch__grid_size"]]))) for r in data])
    lines = [f"ncu --set full --clock-control none --import-source on; command: {command}",
             "one C5 RHS (N=2^20, D=5), kernels in issue order (ncu serialises them)", ""]
    traffic = {}
    for n, (r, lab) in enumerate(zip(data, labs)):
        lines.append(f"[{n}] {lab}   ({short(r[ix['Kernel Name']])})")
        for w in WANT:
            if w in ix:
                lines.append(f"    {w:64s} {r[ix[w]]} {units[ix[w]]}")
        rd = float(r[ix["dram__bytes_read.sum"]]) * TO_BYTES.get(units[ix["dram__bytes_read.sum"]], 1.0)
        wr = float(r[ix["dram__bytes_write.sum"]]) * TO_BYTES.get(units[ix["dram__bytes_write.sum"]], 1.0)
        ms = float(r[ix["gpu__time_duration.sum"]]) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(units[ix["gpu__time_duration.sum"]], 1.0)
        if lab.startswith("pass"):
            traffic[lab] = {"dram_bytes": rd + wr, "read": rd, "write": wr, "ncu_ms": ms}
    out = os.path.join(ROOT, "profiles", f"{tag}_rhs_full_ncu.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    js = os.path.join(ROOT, "profiles", f"{tag}_roofline_traffic.json")
    json.dump({"source": f"profiles/{tag}_rhs_full_ncu.txt ({command}); bytes per launch", "kernels": traffic},
              open(js, "w"), indent=1)
    print(out, js)


if __name__ == "__main__":
    mode, path, tag = sys.argv[1:4]
    command = sys.argv[4] if len(sys.argv) > 4 else ""
    {"launches": launches, "full": full}[mode](path, tag, command)
