"""Summarise a ptxas -v log: kernel (demangled template args), registers, spills."""
import re, sys
cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    if cur and pat in cur:
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m: spill = m.groups()
        m2 = re.search(r"Used (\d+) registers", line)
        if m2:
            args = re.findall(r"ILi(\d+)ELb([01])ELb([01])ELb([01])", cur)
            print(cur[-60:] if not args else args[0], "regs", m2.group(1), "stack/spill st/ld", spill)
