"""Summarise `nvcc -Xptxas -v` output (build log on stdin): kernel, registers, spill bytes."""
import re
import subprocess
import sys

txt = sys.stdin.read()
pat = re.compile(r"Compiling entry function '(\w+)'.*?\n(?:.*?Function properties.*?\n)?\s*(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n.*?Used (\d+) registers", re.S)
flt = sys.argv[1] if len(sys.argv) > 1 else ""
for m in pat.finditer(txt):
    name = m.group(1)
    if flt not in name:
        continue
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    dem = dem.replace("ddl::", "").replace("(CParams)", "").replace("(KParams)", "")
    print(f"{m.group(5):>4} regs  spill st {m.group(3):>5} ld {m.group(4):>5}  {dem}")
