# per-launch sequence of one coarse solve (the second of two): print kernel name + duration in order
import sys
sys.path.insert(0, "/root/repo/tools")
from launches_summary import load
d = load(sys.argv[1])
n = len(d) // 2
for name, v in d[n:]:
    print(f"{v:8.2f}  {name[:70]}")
