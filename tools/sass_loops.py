"""Report loop bodies (backward branches) of a cubin's SASS: size and instruction mix.

    python tools/sass_loops.py file.cubin
"""
import re
import subprocess
import sys
from collections import Counter


def main(path):
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    ins = []
    for line in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr_idx = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, text) in enumerate(ins):
        m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", text)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in addr_idx:
                body = ins[addr_idx[tgt]:i + 1]
                if len(body) < 40:
                    continue
                ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for _, t in body)
                print(f"loop {tgt:#x}..{a:#x}: {len(body)} instructions; top: "
                      + ", ".join(f"{k}={v}" for k, v in ops.most_common(12)))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
