"""Summarise an ncu report: per kernel duration, DRAM bytes/throughput, occupancy, top stalls."""
import csv, subprocess, sys

def summary(rep, regex=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
    r = csv.reader(out)
    hdr = next(r)
    units = dict(zip(hdr, next(r)))
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
    lines = []
    for vals in r:
        d = dict(zip(hdr, vals))
        name = d["Kernel Name"]
        if regex and regex not in name:
            continue
        f = lambda k: float(d.get(k, "0").replace(",", "") or 0) * scale.get(units.get(k, ""), 1.0)
        st = {k: float(v.replace(",", "")) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
              and v.replace(",", "").replace(".", "").isdigit()}
        tot = sum(st.values()) or 1
        stalls = ", ".join(f"{k[33:]}={100*v/tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:6])
        lines.append(f"{name[:60]:60s} {f('gpu__time_duration.sum'):9.4f} ms  dram {f('dram__bytes_read.sum')+f('dram__bytes_write.sum'):8.4f} GB "
                     f"({f('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}%)  regs {d.get('launch__registers_per_thread')}  "
                     f"warps {f('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%  ipc {f('sm__inst_executed.avg.per_cycle_active'):.2f}\n      {stalls}")
    return lines

if __name__ == "__main__":
    for l in summary(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None):
        print(l)
