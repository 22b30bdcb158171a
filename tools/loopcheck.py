"""Static check of the k_lane streaming loop in a built libhist256 (or .o): for each
k_lane instantiation, the innermost loops holding >= 16 ATOMS, their instruction count
and any per-iteration overhead that has cost throughput before (local-memory spills,
R2UR moves of the memory descriptor). usage: python tools/loopcheck.py LIB.so"""
import collections
import re
import subprocess
import sys


def functions(path):
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    cur, body = None, []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if m and cur:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if cur:
        yield cur, body


def back_edges(body):
    for a, t in body:
        if "BRA" not in t:
            continue
        m = re.search(r"0x([0-9a-f]+)\s*$", t)
        if m and int(m.group(1), 16) < a:
            yield int(m.group(1), 16), a


def loops(body, innermost=True):
    edges = list(back_edges(body))
    for tgt, a in edges:
        if innermost and any(tgt <= t2 and a2 < a for t2, a2 in edges if (t2, a2) != (tgt, a)):
            continue
        ins = [x[1] for x in body if tgt <= x[0] <= a]
        if sum("ATOMS" in x for x in ins) >= 16:
            yield tgt, a, ins


def report(path):
    out = []
    for name, body in functions(path):
        if "k_lane" not in name:
            continue
        for tgt, a, ins in loops(body):
            ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for x in ins)
            out.append({"kernel": name, "start": hex(tgt), "len": len(ins), "atoms": ops["ATOMS"],
                        "ldg": ops["LDG"], "r2ur": ops["R2UR"], "local": ops["LDL"] + ops["STL"]})
    return out


if __name__ == "__main__":
    for r in report(sys.argv[1]):
        print(r)
