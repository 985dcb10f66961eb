"""Summarise `nvcc -Xptxas -v` output: registers / spills per kernel.
Usage: python tools/ptxas_regs.py ptxas.txt [filter]"""
import re
import sys

flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and flt in cur:
        print(f"{m.group(1):>4} regs  {cur}")
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur and flt in cur and (m.group(1) != "0" or m.group(2) != "0"):
        print(f"      SPILL {m.group(1)}/{m.group(2)}  {cur}")
