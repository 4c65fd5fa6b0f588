"""Per-kernel counts of the SASS mnemonics that prove which hardware paths the built library uses:
DMMA (FP64 tensor-core MMA), UTMALDG / UBLKCP (TMA tensor and bulk copies), SYNCS (mbarrier), LDGSTS (cp.async),
UTCxMMA / LDTM (tcgen05 -- expected absent: tcgen05 has no f64 kind).  Reads `cuobjdump -sass` of
paper_1707_05594_b200/lib/libtuckerplan_b200.so; prints one line per kernel that contains any of them, then totals."""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1707_05594_b200/lib/libtuckerplan_b200.so"
PATTERNS = collections.OrderedDict([
    ("DMMA", re.compile(r"\bDMMA\.")), ("UTMALDG", re.compile(r"\bUTMALDG")), ("UBLKCP", re.compile(r"\bUBLKCP")),
    ("SYNCS", re.compile(r"\bSYNCS")), ("LDGSTS", re.compile(r"\bLDGSTS")), ("DFMA", re.compile(r"\bDFMA\b")),
    ("UTCMMA", re.compile(r"\bUTC[A-Z]*MMA")), ("LDTM", re.compile(r"\bLDTM")), ("BAR", re.compile(r"\bBAR\.SYNC")),
])


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    counts, current = collections.OrderedDict(), None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            current = m.group(1)
            counts[current] = collections.Counter()
            continue
        if current is None:
            continue
        for name, pat in PATTERNS.items():
            if pat.search(line):
                counts[current][name] += 1
    names = demangle(list(counts))
    total = collections.Counter()
    print("arch: sm_100a   library:", LIB)
    print("%-90s %s" % ("kernel", " ".join("%7s" % n for n in PATTERNS)))
    for fn, c in counts.items():
        total.update(c)
        if not any(c[n] for n in ("DMMA", "UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "UTCMMA", "LDTM")):
            continue
        short = names.get(fn, fn).replace("(anonymous namespace)::", "").replace("tpb::", "").replace("void ", "")
        short = re.sub(r"\(.*", "", short)
        print("%-90s %s" % (short[:90], " ".join("%7d" % c[n] for n in PATTERNS)))
    print("%-90s %s" % ("TOTAL (%d kernels)" % len(counts), " ".join("%7d" % total[n] for n in PATTERNS)))


if __name__ == "__main__":
    main()
