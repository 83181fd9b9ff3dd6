"""Top stall lines of an ncu report's source page: ncu_hot.py report.ncu-rep [n] [kernel-regex]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
if len(sys.argv) > 3:
    cmd += ["--kernel-name", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
if not blocks:
    blocks = [{"name": "?", "rows": rows}]
for b in blocks:
    hdr = b["rows"][0]
    data = [r for r in b["rows"][1:] if len(r) == len(hdr)]
    i_s, i_src, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")

    def f(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    tot = sum(f(r[i_s]) for r in data)
    print(b["name"][:90], "| samples", tot, "| sass", len(data), "| executed", sum(f(r[i_ex]) for r in data))
    # per-reason stall columns (stall_barrier, stall_long_sb, ...), when the report's source page has them
    reasons = [(i, h) for i, h in enumerate(hdr) if h.lower().startswith("stall_") and "not_issued" not in h.lower()]
    for r in sorted(data, key=lambda r: -f(r[i_s]))[:n]:
        why = sorted(((f(r[i]), h) for i, h in reasons if f(r[i]) > 0), reverse=True)[:3]
        print(f"  {f(r[i_s]):7.0f} {100*f(r[i_s])/max(tot,1):5.1f}% {r[i_ex]:>9} {r[i_src][:70]}",
              " ".join(f"{h.split()[0]}={v:.0f}" for v, h in why))
    if reasons:
        tots = sorted(((sum(f(r[i]) for r in data), h) for i, h in reasons), reverse=True)
        print("  stall reasons (all samples):", ", ".join(f"{h.split()[0]} {100*v/max(tot,1):.1f}%" for v, h in tots if v > 0))
    # executed instructions and stall samples by opcode (predicate guards stripped)
    ops = {}
    for r in data:
        toks = [t for t in r[i_src].split() if not t.startswith("@")]
        op = toks[0].split(".")[0] if toks else "?"
        e = ops.setdefault(op, [0.0, 0.0])
        e[0] += f(r[i_ex])
        e[1] += f(r[i_s])
    tex = sum(v[0] for v in ops.values())
    print("  by opcode (executed warp instructions, share; stall samples, share):")
    for op, (ex, sa) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:24]:
        print(f"    {op:10s} {ex:12.0f} {100*ex/max(tex,1):5.1f}%  {sa:7.0f} {100*sa/max(tot,1):5.1f}%")
