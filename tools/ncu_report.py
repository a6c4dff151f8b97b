"""One-paragraph summary of an `ncu --set full` report (.ncu-rep): duration,
DRAM bytes (read + write), throughput figures, occupancy, top stalls."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "Cluster Size", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions", "SM Frequency", "DRAM Frequency"]


def _csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summary(rep):
    rows = _csv(rep, "details")
    hdr = rows[0]
    ni, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ki = hdr.index("Kernel Name")
    kern = rows[1][ki]
    d = {}
    for r in rows[1:]:
        if r[ni] in KEYS and r[ni] not in d:
            d[r[ni]] = (r[vi], r[ui])
    raw = _csv(rep, "raw")
    h, units, v = raw[0], raw[1], raw[-1]
    def val(name):
        i = h.index(name)
        x = float(v[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return x * scale
    dram = None
    try:
        dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    except Exception:
        pass
    stalls = []
    for name, x in zip(h, v):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(x), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    return kern, d, dram, stalls[:5]


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        kern, d, dram, stalls = summary(rep)
        print(f"== {rep}\nkernel: {kern[:160]}")
        for k in KEYS:
            if k in d:
                print(f"  {k}: {d[k][0]} {d[k][1]}")
        if dram is not None:
            print(f"  dram bytes (read+write): {dram:.4e}")
        print("  top stalls (warps per issue): " + ", ".join(f"{n}={x:.2f}" for x, n in stalls))
