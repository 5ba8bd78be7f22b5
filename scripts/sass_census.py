"""Blackwell instruction census of every kernel in libgfb200.so (and of a
generated row-fused / elementwise kernel): counts of the SASS mnemonics that
prove the sm_100a paths (B200_PROFILING.md "What proves a Blackwell-native
kernel"): UTC*MMA = tcgen05.mma, UTMALDG = TMA tensor load, UBLKCP =
cp.async.bulk, LDTM / STTM = tcgen05.ld / st, LDGSTS = cp.async."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1801_08058_b200", "libgfb200.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "UTCOMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "LDGSTS", "HMMA",
        "SHFL", "DFMA", "MUFU"]


def census(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op.startswith(k):
                    kernels[cur][k] += 1
    return kernels


def main():
    paths = [LIB] + sys.argv[1:]
    for p in paths:
        print(f"# {os.path.relpath(p, ROOT)}")
        for name, c in census(p).items():
            demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            cols = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
            print(f"{demangled[:90]:90s} {cols}")


if __name__ == "__main__":
    main()
