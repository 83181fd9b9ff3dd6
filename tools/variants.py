"""A/B timing of kernel variants on one box: variants.py ENVVAR v1,v2,... CFG[,CFG] [reps].
Each variant runs in a fresh subprocess (the env var is read once per process)."""
import json
import os
import subprocess
import sys

var, vals, cfgs = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
reps = sys.argv[4] if len(sys.argv) > 4 else "5"
here = os.path.dirname(os.path.abspath(__file__))
for rnd in range(2):
    for v in vals:
        env = dict(os.environ, **{var: v})
        out = subprocess.run([sys.executable, os.path.join(here, "phase_times.py"), cfgs, reps], env=env,
                             capture_output=True, text=True)
        for line in out.stdout.splitlines():
            name, js = line.split(" ", 1)
            d = json.loads(js)
            print(f"round {rnd} {var}={v} {name}: sweep/colour {d['sweep_us_per_colour']:.2f} us, "
                  f"{d['sweep_tflops']:.2f} TFLOP/s, apply {d['apply_us']:.1f} us ({d['apply_GBps']:.0f} GB/s), "
                  f"defect+R {d['defect_restrict_us']:.1f}, prolong {d['prolong_us']:.1f}, coarse {d['coarse_us']:.1f}, "
                  f"iter {d['iter_us']:.1f} us", flush=True)
        if out.returncode:
            print(out.stderr[-2000:])
