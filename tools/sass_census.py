"""SASS instruction census of the built kernels (cuobjdump -sass on build/apx/*.o): per kernel,
the counts of the instructions that prove the execution units used -- tcgen05 MMA (UTCHMMA /
UTCQMMA...), TMA (UTMALDG / UTMASTG), TMEM loads (LDTM), tensor-core barriers (UTCBAR), DMMA,
FFMA2 / FFMA / DFMA, shared loads (LDS*) -- written to profiles/r02_sass_census.txt."""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "UTCBAR", "DMMA", "HMMA",
        "FFMA2", "FFMA", "DFMA", "DADD", "DMUL", "LDS", "STS", "LDG", "STG", "SHFL", "SYNCS"]


def census(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(1).split(".")[0]
            for k in KEYS:
                if op == k:
                    per[cur][k] += 1
    return per


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


def main():
    lines = []
    for obj in sorted(glob.glob(os.path.join(ROOT, "build", "apx", "*.o"))):
        per = census(obj)
        if not per:
            continue
        lines.append(f"== {os.path.basename(obj)}")
        names = demangle(list(per))
        for (raw, cnt), name in zip(per.items(), names):
            if not cnt:
                continue
            short = re.sub(r"\(.*", "", name)[:110]
            lines.append(f"  {short}: " + ", ".join(f"{k} {cnt[k]}" for k in KEYS if cnt[k]))
    text = "\n".join(lines) + "\n"
    dst = os.path.join(ROOT, "profiles", "r02_sass_census.txt")
    open(dst, "w").write("# cuobjdump -sass census of build/apx/*.o (tools/sass_census.py)\n" + text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
