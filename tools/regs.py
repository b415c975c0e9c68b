"""Registers / spills per kernel instantiation of libsystec.so (cuobjdump -res-usage)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2406_09266_b200/libsystec.so"
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout.splitlines()
name = None
for line in out:
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
    if m and name:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        if pat is None or pat.search(dem):
            print(f"REG={m.group(1):>3} STACK={m.group(2):>3} LOCAL={m.group(4):>3}  {dem[:110]}")
        name = None
