"""Markdown summary of the Blackwell instructions in the built library's SASS (the proof
that the GEMMs are tcgen05 / TMA / TMEM kernels): per kernel, counts of UTCHMMA (tcgen05.mma),
UTCBAR (tcgen05.commit), UTMALDG / UTMASTG (TMA loads / stores), LDTM (tcgen05.ld), HMMA
(mma.sync), plus an excerpt of one kernel.  usage: python tools/sass_summary.py > profiles/..."""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2303_06318_b200/libted_b200.so"
EXCERPT = sys.argv[2] if len(sys.argv) > 2 else "grouped_gemm_kernelILb1ELb1ELi4ELb1E"
MN = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "LDTM", "HMMA", "UTCATOMSWS"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)[1:]
print(f"# SASS of `{LIB}` (cuobjdump -sass)\n")
print("grouped_gemm_kernel<A_MN, B_MN, EPI, PAIR>: EPI 0 store, 1 bias, 2 bias+GELU, 3 dGELU, "
      "4 AdamW; PAIR = the cta_group::2 variant (`.2CTA` forms below).  UTCHMMA = "
      "tcgen05.mma, UTCBAR = tcgen05.commit, UTMALDG / UTMASTG = TMA tensor load / store, "
      "LDTM = tcgen05.ld, UTCATOMSWS = TMEM alloc / dealloc, HMMA = mma.sync (the routing "
      "kernels' small products).  Counts are static instruction counts.\n")
print("| kernel (demangled template args) | " + " | ".join(MN) + " |")
print("|---|" + "---|" * len(MN))


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"ted::\(anonymous namespace\)::", "", d)
    return d.split("(")[0]


for f in funcs:
    name = f.split("\n", 1)[0].strip()
    cnt = [len(re.findall(r"\b" + m + r"[\.\s]", f)) for m in MN]
    if any(cnt):
        print(f"| `{short(name)}` | " + " | ".join(str(c) for c in cnt) + " |")
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if EXCERPT in name:
        print(f"\n## Excerpt: `{short(name)}`\n\n```")
        for l in f.split("\n"):
            if re.search(r"UTCHMMA|UTMALDG|UTMASTG|LDTM|UTCBAR|UTCATOMSWS|ELECT", l):
                print(re.sub(r"\s+", " ", l.strip()))
        print("```")
        break
