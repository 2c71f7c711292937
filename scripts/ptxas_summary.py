"""One line per kernel from the last build's ptxas -v log: registers, stack, spills."""
import re, subprocess, sys, os
log = open(os.path.join(os.path.dirname(__file__), "..", "paper_2605_00830_b200", "csrc", "ptxas.log")).read()
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip().split("(")[0]
        cur = cur.replace("fg::", "").replace("unsigned char", "u8").replace("unsigned short", "u16")
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        stack = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:60s} regs {m.group(1):>4s} stack {stack[0]:>3s} spill st/ld {stack[1]}/{stack[2]}")
        cur = None
