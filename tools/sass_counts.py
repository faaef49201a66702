"""Per-kernel SASS instruction counts of the built library (evidence that the tile movement is
Blackwell-native: UTMALDG = TMA tensor loads, UBLKCP = bulk copies, STTM / LDTM = tcgen05 TMEM
stores / loads, SYNCS = mbarrier ops, plus shuffles, fp64 FMAs and atomics).

usage: python tools/sass_counts.py [lib.so] > profiles/rNN_sass_counts.txt"""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1701_04900_b200/lib/libasyflexa.so"
OPS = ["UTMALDG", "UBLKCP", "STTM", "LDTM", "UTCATOMSWS", "SYNCS", "SHFL", "DFMA", "DADD", "REDG", "ATOMG",
       "ATOMS", "LDS", "STS", "LDG", "STG", "MEMBAR", "FENCE", "NANOSLEEP"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.strip().split("\n")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = {op: 0 for op in OPS}
            funcs[cur]["total"] = 0
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.\S+)?", line)
        if not m:
            continue
        op = m.group(2)
        funcs[cur]["total"] += 1
        for o in OPS:
            if op == o:
                funcs[cur][o] += 1
    names = [n for n in funcs if n.startswith("_ZN3asy")]
    pretty = demangle(names)
    print("# SASS instruction counts per kernel: cuobjdump -sass %s (sm_100a)" % LIB)
    print("%-78s %7s " % ("kernel", "total") + " ".join("%7s" % o for o in OPS))
    for n, p in zip(names, pretty):
        p = re.sub(r"\(.*\)$", "", p).replace("asy::", "")
        f = funcs[n]
        print("%-78s %7d " % (p[:78], f["total"]) + " ".join("%7d" % f[o] for o in OPS))


if __name__ == "__main__":
    main()
