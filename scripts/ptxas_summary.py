"""Registers / spills per kernel from the ptxas -v logs in build/ctqw."""
import glob
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
for path in sorted(glob.glob("build/ctqw/*.ptxas.log")):
    log = open(path).read()
    for b in re.split(r"ptxas info    : Compiling entry function '", log)[1:]:
        name = b.split("'")[0]
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        if pat and pat not in dem:
            continue
        regs = re.search(r"Used (\d+) registers", b)
        sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", b)
        short = re.sub(r"\(.*", "", dem.replace("ctqw::", "").replace("b4::", ""))
        print(f"{short:70s} regs {regs.group(1) if regs else '?':>4s} spill st/ld {sp.groups() if sp else ''}")
