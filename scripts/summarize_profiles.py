"""Turn gpurun_out/{launches.csv,prof_top.ncu-rep,bench_full.log} into profiles/ summaries."""
import collections, csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out"); P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(P, exist_ok=True)
# 1) launch list
rows = [r for r in csv.reader(open(os.path.join(G, "launches.csv"))) if len(r) > 10]
hdr = rows[0]; rows = rows[1:]
iI, iK, iM, iV = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
per = collections.defaultdict(dict)
for r in rows:
    per[int(r[iI])][r[iM]] = float(r[iV].replace(",", ""))
    per[int(r[iI])]["name"] = r[iK]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in sorted(per):
    d = per[i]
    n = d["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    a = agg[n]; a[0] += 1; a[1] += d.get("gpu__time_duration.sum", 0); a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
tot = sum(v[1] for v in agg.values())
lines = [f"# ncu launch list ({tag}): python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu (C3)",
         "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
         "# per-launch times are cold-cache and serialised: compare SHARES, not absolutes",
         f"{'kernel':58s} {'launches':>8s} {'total_ms':>9s} {'share':>6s} {'avg_us':>9s} {'dram_GB/launch':>14s}"]
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{n[:58]:58s} {c:8d} {t/1e6:9.3f} {100*t/tot:5.1f}% {t/c/1e3:9.1f} {b/c/1e9:14.4f}")
open(os.path.join(P, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:14]))
# 2) full capture summary of the top kernels
rep = os.path.join(G, "prof_top.ncu-rep")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out); hdr = next(r); next(r)
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
traffic = {}
txt = [f"# ncu --set full --clock-control none --import-source on ({tag}), C3 bench, steady-state launches"]
for vals in r:
    d = dict(zip(hdr, vals))
    name = d["Kernel Name"].split("(")[0]
    st = {k: float(v.replace(",", "")) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled")
          and not k.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()}
    s = sum(st.values()) or 1
    txt.append(f"\n## {name}")
    for k in want:
        txt.append(f"  {k:62s} {d.get(k, '')}")
    txt.append("  top stall reasons: " + ", ".join(f"{k[33:]}={100*v/s:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]))
    b = float(d["dram__bytes_read.sum"].replace(",", "")) + float(d["dram__bytes_write.sum"].replace(",", ""))
    unit = d.get("dram__bytes_read.sum", "")
    # xsweep_kernel<P, INLINE, RHO, FMA>: the fused-moment variant is x sweep 1
    targs = d["Kernel Name"].split("<", 1)[-1].split(">")[0].split(",")
    rho = len(targs) > 2 and ("1" in targs[2] or "true" in targs[2])
    key = (("x_sweep_1" if rho else "x_sweep_2") if "xsweep" in name
           else "v_sweep" if "vsweep" in name else name)
    traffic.setdefault(key, b)
open(os.path.join(P, f"{tag}_ncu_full.txt"), "w").write("\n".join(txt) + "\n")
# units: ncu raw csv reports dram bytes in the unit row; convert GB -> bytes if needed
units_row = out[1]
tr = {}
for k, v in traffic.items():
    tr[k] = v * (1e9 if v < 1e4 else 1.0)
json.dump({"C3": {"x_sweep_1": tr.get("x_sweep_1"), "x_sweep_2": tr.get("x_sweep_2"), "v_sweep": tr.get("v_sweep")}},
          open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(P, f"{tag}_ncu_full.txt")).read()[:3000])
# 3) bench line
b = open(os.path.join(G, "bench_full.log")).read().strip().splitlines()[-1]
open(os.path.join(P, f"{tag}_bench_C3.json"), "w").write(b + "\n")
