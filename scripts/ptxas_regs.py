"""Registers / spills per softmax pipeline instantiation from the ptxas logs (build aid)."""
import glob
import re
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "paper_2412_00408_b200/build"
for fn in sorted(glob.glob(f"{d}/*.ptxas.log")):
    for blk in open(fn).read().split("ptxas info    : Compiling entry function")[1:]:
        name = blk.split("'")[1]
        mm = re.search(r"\d(softmax_[a-z0-9_]+?)ILNS_8SmKernelE(\d)E(?:Lb(\d)E)?(?:Li(\d+)E)?", name)
        if not mm:
            continue
        sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", blk)
        r = re.search(r"Used (\d+) registers", blk)
        print(f"{fn.split('/')[-1]:28s} {mm.group(1):18s} K{mm.group(2)} cl{mm.group(3)} KC{mm.group(4)} "
              f"regs {r.group(1)} spill {sp.group(1)}/{sp.group(2)}")
