"""Dev helper: summarise `nvcc -Xptxas -v` per kernel (registers, spills, smem)."""
import re, subprocess, sys
cmd = ["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
       "-lineinfo", "--fmad=false", "-Iinclude", "-Xptxas", "-v", "-c", "-o", "/dev/null",
       sys.argv[1] if len(sys.argv) > 1 else "paper_1512_08017_b200/csrc/k_power_sums.cu"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur: spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{m.group(1):>4} regs  spill st/ld {spill[0]}/{spill[1]:<5} {cur[:90]}")
