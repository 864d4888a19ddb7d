"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked).

    python tools/make_profiles.py <round-tag> <launches.csv> <full.ncu-rep[,more.ncu-rep]> [config]
"""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary

tag, launches, rep = sys.argv[1:4]
cfg = sys.argv[4] if len(sys.argv) > 4 else "C3"
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
os.makedirs(out, exist_ok=True)
txt = subprocess.check_output([sys.executable, os.path.join(os.path.dirname(__file__), "launches.py"),
                               launches, "40"], text=True)
with open(os.path.join(out, "%s_launches_%s.txt" % (tag, cfg)), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, command: "
            "python bench.py --steps 2 --warmup 1 --no-cpu-baseline (config %s)\n"
            "# per-launch times are cold-cache and serialised: compare SHARES, not absolutes\n"
            "# total_us  share  launches  us_per_launch  kernel\n" % cfg)
    f.write(txt)
summ = [d for r in rep.split(",") for d in summary(r)]
with open(os.path.join(out, "%s_ncu_full_%s.json" % (tag, cfg)), "w") as f:
    json.dump(summ, f, indent=1)
traffic = {}
for d in summ:
    def val(k):
        v, _, u = d[k].partition(" ")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return float(v.replace(",", "")) * mult
    name = d["kernel"].split("::")[-1]
    traffic[name] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
with open(os.path.join(out, "traffic_%s.json" % cfg), "w") as f:
    json.dump(dict(traffic, _source="%s ncu --set full (dram__bytes_read.sum + dram__bytes_write.sum per launch)" % tag), f, indent=1)
print(txt)
print(json.dumps(traffic))
