"""Count the SASS instructions of a kernel's per-entry loop (the innermost
backward branch around the B-row gathers), by opcode.  Build aid: compare
kernel variants before spending GPU time.

    python tools/hotloop.py [lib] 'mttkrp_sym_kernel_occILi3ELi8ELi1ELi4ELb1'
"""
import collections
import re
import subprocess
import sys

ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))


def functions(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
        if cur and m:
            body.append((int(m.group(1), 16), m.group(2)))
    if cur:
        yield cur, body


def hot_loop(body):
    """Smallest backward-branch loop that contains a 128- or 256-bit global gather."""
    best = None
    for addr, ins in body:
        m = re.search(r"BRA (?:`\()?\.?L?_?x?_?(0x[0-9a-f]+|\d+)", ins)
        if not m:
            continue
        try:
            tgt = int(m.group(1), 16)
        except ValueError:
            continue
        if tgt >= addr:
            continue
        loop = [(a, i) for a, i in body if tgt <= a <= addr]
        if any(("LDG.E.128" in i or ".256" in i and "LDG" in i) for _, i in loop) and (best is None or len(loop) < len(best)):
            best = loop
    return best or []


def main():
    args = sys.argv[1:]
    lib = args.pop(0) if args and args[0].endswith(".so") else f"{ROOT}/paper_2406_09266_b200/libsystec.so"
    pat = args[0] if args else "mttkrp_sym_kernel_occILi3ELi8ELi1ELi4ELb1"
    for name, body in functions(lib):
        if pat not in name:
            continue
        loop = hot_loop(body)
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0].split(".")[0] for _, i in loop)
        print(f"{name}: {len(body)} instructions, hot loop {len(loop)}")
        print("   " + ", ".join(f"{o} {n}" for o, n in ops.most_common()))


if __name__ == "__main__":
    main()
