"""Opcode histogram of selected kernels in libparplan_cuda.so (cuobjdump -sass):
whole kernel and the hottest loop (the instructions between the first and the
last occurrence of the kernel's key opcode).
  python tools/sass_histogram.py > profiles/r02_sass_opcodes.txt"""
import collections
import os
import re
import subprocess

SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1802_04924_b200",
                  "libparplan_cuda.so")
KERNELS = [("mp_fold_kernel<6>", "_ZN2pp14mp_fold_kernelILi6EEEvPKNS_6MpFoldEill", "VIADDMNMX"),
           ("mp_chain_kernel<6,7>", "_ZN2pp15mp_chain_kernelILi6ELi7EEEvPKNS_6MpFoldEii", "VIADDMNMX"),
           ("mp64_fold_kernel", "_ZN2pp16mp64_fold_kernelEPKNS_8Mp64FoldEi", "DADD"),
           ("mp_prep_kernel", "_ZN2pp14mp_prep_kernelEPKNS_6MpFoldEi", "LDG"),
           ("build_tables_kernel", "_ZN2pp19build_tables_kernelENS_9BuildArgsE", "IMAD")]
OP = re.compile(r"^\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?")

for label, sym, key in KERNELS:
    out = subprocess.run(["cuobjdump", "-sass", "-fun", sym, SO], capture_output=True, text=True).stdout
    ops = []
    for line in out.splitlines():
        m = OP.match(line)
        if m:
            ops.append(m.group(2) + (m.group(3) or ""))
    if not ops:
        print(f"== {label}: not found")
        continue
    idx = [i for i, o in enumerate(ops) if o.startswith(key)]
    print(f"== {label} ({sym}): {len(ops)} instructions")
    whole = collections.Counter(o.split(".")[0] for o in ops)
    print("   whole kernel:", ", ".join(f"{k} {v}" for k, v in whole.most_common(14)))
    if idx:
        hot = collections.Counter(ops[idx[0]: idx[-1] + 1])
        n = idx[-1] + 1 - idx[0]
        print(f"   hot region ({n} instructions between the first and last {key}):")
        for k, v in hot.most_common(12):
            print(f"      {k:28s} {v:6d}  {v / n:6.1%}")
    bulk = [o for o in ops if o.startswith(("UBLKCP", "UTMALDG", "SYNCS"))]
    print("   async copy / mbarrier ops:", ", ".join(f"{k} {v}" for k, v in collections.Counter(bulk).most_common()))
