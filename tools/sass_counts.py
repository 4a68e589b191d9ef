"""Per-kernel SASS instruction counts of the shipped library (cuobjdump -sass):
the bulk-copy / prefetch / async-copy / spill / FP64 / shuffle mnemonics that
show what each hot kernel actually does.  usage: python tools/sass_counts.py [lib]"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2306_11665_b200/libsumfac_b200.so"
KEYS = ["UBLKCP", "UBLKPF", "LDGSTS", "SYNCS", "STL", "LDL", "DFMA", "DMUL", "DADD", "MUFU",
        "SHFL", "LDS", "STS", "LDG", "STG", "BAR", "DMMA"]
HOT = ["euler_cart_own_kernel", "euler_cart_sync_kernel", "euler_cartesian_kernel",
       "euler_cart_node_kernel", "euler_cart_n2_kernel", "euler_cart_n3_kernel", "euler_modal_kernel", "hadamard_rowsum_fixed_kernel",
       "hadamard_rowsum_generic_kernel", "burgers_rk4"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m:
        funcs[cur][m.group(1)] += 1
print("kernel (demangled prefix) | " + " | ".join(KEYS) + " | total")
for name, c in funcs.items():
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    if not any(h in dem for h in HOT):
        continue
    short = dem.replace("(anonymous namespace)::", "").split("(")[0].replace("sfb::", "")
    print(f"{short} | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + f" | {sum(c.values())}")
