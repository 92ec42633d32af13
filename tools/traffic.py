"""ncu-measured DRAM traffic per bench workload -> profiles/r2/traffic_r2.json (read by
bench.py as the roofline `traffic` field).

  on the GPU box:  python tools/traffic.py run C2 C3 ...     (ncu, one process per workload)
  here:            python tools/traffic.py parse            (gpurun_out/tr_*.csv -> json)

Each workload runs `bench.py --ncu --steps 2 --warmup 3`: 3 warm-up + 2 timed + 2 split
steps = 7 identical steps, every kernel launch profiled with dram__bytes_read.sum and
dram__bytes_write.sum (cold-cache, serialised replay).  Traffic per step = all launches / 7."""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = 7
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def run(workloads):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for w in workloads:
        log = os.path.join(ROOT, "gpurun_out", f"tr_{w}.csv")
        cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--csv", "--log-file", log,
               sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, "--steps", "2",
               "--warmup", "3", "--ncu"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        print(w, "rc", r.returncode, flush=True)


def parse():
    out = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "tr_*.csv"))):
        w = os.path.basename(path)[3:-4]
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
        if not rows:
            continue
        hdr = rows[0]
        ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
        kern = {}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                 "msecond": 1e-3}
        for r in rows[1:]:
            name = r[ki].split("(")[0].split("<")[0].replace("(anonymous namespace)::", "")
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
            d = kern.setdefault(name, {"read": 0.0, "write": 0.0, "time_s": 0.0, "launches": 0})
            if r[mi].startswith("dram__bytes_read"):
                d["read"] += v
                d["launches"] += 1
            elif r[mi].startswith("dram__bytes_write"):
                d["write"] += v
            else:
                d["time_s"] += v
        per = {k: {"dram_bytes_per_step": (d["read"] + d["write"]) / STEPS,
                   "read_per_step": d["read"] / STEPS, "write_per_step": d["write"] / STEPS,
                   "launches_per_step": d["launches"] / STEPS,
                   "ncu_time_share": 0.0, "ncu_us_per_step": 1e6 * d["time_s"] / STEPS}
               for k, d in kern.items()}
        tt = sum(d["time_s"] for d in kern.values()) or 1.0
        for k, d in kern.items():
            per[k]["ncu_time_share"] = d["time_s"] / tt
        top = max(per, key=lambda k: per[k]["ncu_time_share"])
        out[w] = {"dram_bytes_per_step": sum(p["dram_bytes_per_step"] for p in per.values()),
                  "dominant_kernel": top,
                  "dominant_bytes_per_launch": per[top]["dram_bytes_per_step"] / max(per[top]["launches_per_step"], 1),
                  "kernels": per,
                  "source": f"ncu --metrics {METRICS} --clock-control none, bench.py --workload {w} "
                            f"--steps 2 --warmup 3 --ncu ({STEPS} steps), {os.path.basename(path)}"}
    dst = os.path.join(ROOT, "profiles", "r2", "traffic_r2.json")
    # merge: workloads not re-captured keep their earlier entries
    merged = json.load(open(dst)) if os.path.exists(dst) else {}
    merged.update(out)
    json.dump(merged, open(dst, "w"), indent=1, sort_keys=True)
    for w, d in out.items():
        print(f"{w:10s} {d['dram_bytes_per_step'] / 1e9:7.3f} GB/step  top {d['dominant_kernel']} "
              f"{d['kernels'][d['dominant_kernel']]['ncu_time_share']:.2f}")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2:])
    else:
        parse()
