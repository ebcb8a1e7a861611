"""Print registers / shared / local memory per kernel of libbsct.so (cuobjdump -res-usage)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2005_13471_b200/libbsct.so"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
name = None
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"REG:(\d+).*SHARED:(\d+) LOCAL:(\d+)", line)
    if m and name and re.search(pat, name):
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"bsct::|cplx_of<(\w+)>::type", r"\1", dem)
        print(f"REG {m.group(1):>4} SMEM {m.group(2):>6} LOCAL {m.group(3):>4}  {dem[:150]}")
