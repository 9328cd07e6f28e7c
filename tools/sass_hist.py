"""SASS instruction histogram per hot kernel of liboomb.so (cuobjdump -sass): proves the tcgen05 / TMA
instructions (UTCHMMA / UTCQMMA, LDTM / STTM, UTMALDG / UTMASTG / UTMAREDG, UBLKCP) and shows each
kernel's instruction mix. Usage: python tools/sass_hist.py [lib.so] > profiles/rNN_sass_hist.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2602_02108_b200/liboomb.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern = None
hist = collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and kern:
        hist[kern][m.group(1)] += 1
HOT = ("attn_fwd_tc4", "attn_bwd_dq", "attn_bwd_dkdv", "score_stats", "score_vote", "topk_kernel", "append_kernel",
       "accumulate_grads_kernel", "bwd_prep")
KEY = ("UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "UBLKRED",
       "SYNCS", "MUFU", "FFMA", "FMUL", "FADD", "F2FP", "LDS", "STS", "LDG", "STG", "BAR", "WARPSYNC")
print(f"# SASS instruction histogram (`cuobjdump -sass {lib}`)\n")
print("Instruction counts are static (per kernel body), not dynamic. tcgen05.mma = UTCHMMA/UTCQMMA, "
      "tcgen05.ld/st = LDTM/STTM, TMA = UTMALDG (load) / UTMASTG (store) / UTMAREDG (reduce-add), "
      "mbarrier = SYNCS.\n")
print("| kernel | " + " | ".join(KEY) + " | total |")
print("|---|" + "---|" * (len(KEY) + 1))
dem = dict(zip(hist, subprocess.run(["c++filt"], input="\n".join(hist), capture_output=True,
                                    text=True).stdout.splitlines()))


def pretty(k):
    d = dem.get(k, k).replace("(anonymous namespace)::", "")
    d = re.sub(r"\(.*$", "", d)  # drop the argument list
    return d.replace("oomb::", "").replace("__nv_bfloat16", "bf16")


rows = sorted((pretty(k), k) for k in hist if any(h in pretty(k) for h in HOT))
for name, k in rows:
    c = hist[k]
    print(f"| `{name}` | " + " | ".join(str(c.get(x, 0)) for x in KEY) + f" | {sum(c.values())} |")
print("\nTop 25 mnemonics of each tcgen05 kernel:\n")
for name, k in rows:
    if hist[k].get("UTCHMMA", 0) == 0:
        continue
    print(f"* **{name}**: " + ", ".join(f"{m} {n}" for m, n in hist[k].most_common(25)))
