"""Developer probe: registers/spills per kernel from the ptxas -v logs."""
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
for log in sys.argv[2:] or ["build/obj/kernels.ptxas.log", "build/obj/pcg.ptxas.log"]:
    name = None
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        m = re.search(r"Used (\d+) registers", line)
        if m and name and pat in name:
            print(m.group(1), name[:110])
