"""Static SASS mix of the fast kernel's TMEM block loop (MODE 2: the loop
holding the STTM.x4 survivor stores), per 4-stage block, split by pipe.

    python tools/loop_mix.py [object-or-library] [kernel-name-substring]
"""
import collections
import re
import subprocess
import sys

ALU = {"VIADDMNMX.S16x2", "IADD3", "PRMT", "LOP3.LUT", "ISETP.GE.AND", "ISETP.NE.AND", "LEA.HI", "LEA", "SHF.R.U32.HI",
       "SHF.L.U32", "SEL", "VIMNMX.S16x2", "VIMNMX3.S16x2", "IADD3.X", "FLO.U32", "SHF.R.W.U32"}
FMAH = {"VIADD.16x2", "IMAD", "IMAD.IADD", "IMAD.MOV.U32", "IMAD.X", "IMAD.SHL.U32", "IMAD.WIDE.U32", "IMAD.U32",
        "IMAD.HI.U32", "IMAD.WIDE"}


def main():
    obj = sys.argv[1] if len(sys.argv) > 1 else "paper_2011_09337_b200/build/vd_fast_k7.o"
    pat = sys.argv[2] if len(sys.argv) > 2 else "CodeBILi7ELi2ELj121ELj91ELj0ELj0EEELi16ELb1ELb0ENS0_7NoPunct"
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", txt)
    f = next(x for x in funcs if pat in x.split("\n")[0])
    ins = [(int(a, 16), t.strip()) for a, t in re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", f)]
    sttm = [i for i, (_, t) in enumerate(ins) if "STTM.x4" in t]
    addr_idx = {a: i for i, (a, _) in enumerate(ins)}
    best = None  # innermost backward branch whose loop holds both STTM.x4 blocks
    for j, (a, t) in enumerate(ins):
        m = re.search(r"BRA\S*\s+(?:\S+,\s*)?0x([0-9a-f]+)", t)
        if not m:
            continue
        lo = addr_idx.get(int(m.group(1), 16))
        if lo is not None and lo <= sttm[0] and j >= sttm[-1] and (best is None or j - lo < best[1] - best[0]):
            best = (lo, j)
    lo, j = best
    body = [t for _, t in ins[lo:j + 1]]
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
    blocks = len(sttm)
    alu = sum(v for k, v in ops.items() if k in ALU)
    fma = sum(v for k, v in ops.items() if k in FMAH)
    print(f"loop: {len(body)} instrs over {blocks} blocks -> {len(body) / blocks:.1f} per block; "
          f"alu {alu / blocks:.1f}, fmaheavy {fma / blocks:.1f}, other {(len(body) - alu - fma) / blocks:.1f}")
    print(" ".join(f"{k}:{v}" for k, v in ops.most_common()))


if __name__ == "__main__":
    main()
