"""Registers / spills per kernel from the ptxas -v log of kernels.cu."""
import re, sys
cur = None
out = {}
for line in open(sys.argv[1] if len(sys.argv) > 1 else "build/obj/ptxas_kernels.txt"):
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1); out[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        out[cur]["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        out[cur]["regs"] = int(m.group(1))
for k, v in out.items():
    m = re.search(r"spmv_block_kernelI([fd])Li(\d+)ELb([01])ELb([01])", k)
    name = f"block {m.group(1)} cfg{m.group(2)} combine={m.group(3)} ident={m.group(4)}" if m else k[-60:]
    print(f"{name:45s} regs {v.get('regs')}  spill st/ld {v.get('spill')}")
