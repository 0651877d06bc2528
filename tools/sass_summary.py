"""Per-kernel SASS opcode summary of the built library (committed per round as
evidence of the instruction mix: tcgen05 MMA / TMEM / bulk-copy / packed FP32).

    python tools/sass_summary.py [paper_2504_11681_b200/libturbofno.so] > profiles/rNN/sass_summary.txt
"""
import collections
import re
import subprocess
import sys

KEY = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UBLKPF", "SYNCS",
       "FFMA2", "FADD2", "FMUL2", "FFMA", "HMMA", "LDS", "STS", "LDG", "STG", "SHFL", "BAR", "LDSM"]


def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    kern, counts = None, collections.defaultdict(collections.Counter)
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if kern and m:
            counts[kern][m.group(1)] += 1
    fam = collections.defaultdict(lambda: [0, collections.Counter()])
    for k, c in counts.items():
        name = re.sub(r"^void |<.*$|\(.*$", "", k.replace("(anonymous namespace)::", "")).replace("tfno::", "")
        fam[name][0] += 1
        fam[name][1].update(c)
    print(f"SASS opcode counts per kernel family (static instruction counts summed over template instances) of {path}")
    print("family".ljust(28) + "inst".rjust(5) + "".join(k.rjust(9) for k in KEY))
    for name in sorted(fam):
        n, c = fam[name]
        print(name[:27].ljust(28) + str(n).rjust(5) + "".join(str(c.get(k, 0)).rjust(9) for k in KEY))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2504_11681_b200/libturbofno.so")
