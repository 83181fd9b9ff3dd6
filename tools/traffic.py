"""DRAM traffic per launch of the dominant kernel from `ncu --set full` reports (one per bench config).

    python tools/traffic.py C2=gpurun_out/ncu_C2.ncu-rep C3=... > profiles/schwarz_traffic.json

Per config: mean over the captured launches of dram__bytes_read.sum + dram__bytes_write.sum (cold cache:
ncu flushes caches between replays), plus the launches' names and durations.
"""
import csv
import io
import json
import subprocess
import sys


def rows(rep):
    if rep.endswith(".csv"):                # `ncu -i rep --page raw --csv` saved on the GPU box
        out = open(rep).read()
        out = out[out.index('"ID"'):] if '"ID"' in out else out
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                             capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return hdr, units, r[2:]


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return float(v.replace(",", "")) * f.get(unit, 1)


res = {}
for arg in sys.argv[1:]:
    cfg, rep = arg.split("=", 1)          # cfg=path[@profile name for the source note]
    rep, _, note = rep.partition("@")
    hdr, units, data = rows(rep)
    i_n = hdr.index("Kernel Name")
    i_r, i_w, i_t = (hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"))
    per = [(d[i_n], scale(d[i_r], units[i_r]) + scale(d[i_w], units[i_w]), scale(d[i_t], units[i_t])) for d in data]
    res[cfg] = {"kernel": sorted({p[0][:90] for p in per}),
                "dram_bytes_per_launch": sum(p[1] for p in per) / len(per),
                "launches_captured": len(per),
                "cold_us_per_launch": [round(p[2], 2) for p in per],
                "source": f"ncu --set full --clock-control none (profiles/{note or 'ncu_traffic_' + cfg + '_r01.txt'}); "
                          f"cold cache, mean over the captured launches"}
print(json.dumps(res, indent=1))
