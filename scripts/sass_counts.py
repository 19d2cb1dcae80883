"""Per-kernel SASS instruction counts of libchfsi_b200.so (cuobjdump -sass): the
evidence that the filter kernels run on the FP64 tensor pipe (DMMA.8x8x4), load
operands by TMA (UTMALDG) and synchronise on mbarriers (SYNCS), with no DFMA in the
main loop. Usage: python scripts/sass_counts.py > profiles/r02/sass_counts.txt"""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1305_5120_b200/_lib/libchfsi_b200.so"
OPS = ["DMMA", "UTMALDG", "SYNCS", "DFMA", "DADD", "DMUL", "LDS", "LDG", "STG", "BAR"]
# zgemm_tma_kernel<BM, BN, WM, WN, STAGES, EPI, WARPS_M?, MUL, SUMS> template args
EPI = {0: "store", 1: "filter", 2: "partial"}

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", sass)
print(f"# {LIB}: SASS opcode counts per kernel (cuobjdump -sass)")
print("# kernel | " + " | ".join(OPS))
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if "zgemm_tma_kernel" not in name and "zgemv" not in name:
        continue
    counts = {op: len(re.findall(r"\b" + op + r"[\.\s]", b)) for op in OPS}
    m = re.search(r"zgemm_tma_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d)E", name)
    if m:
        bm, bn, wm, wn, st, epi, _, mul, sums = (int(x) for x in m.groups())
        label = (f"zgemm_tma<{bm}x{bn}, warp {wm}x{wn}, {st} stages, epi={EPI.get(epi, epi)}, "
                 f"{'3M' if mul == 3 else '4 products'}"
                 f"{['', ', sum planes', ', B-sum plane only + packed tail block'][sums]}>")
    else:
        label = name[:80]
    print(label + " | " + " | ".join(str(counts[op]) for op in OPS))
