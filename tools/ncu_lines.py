"""Attribute an ncu source-page (SASS) export of kernel 3 to CUDA source lines
and warp roles (dev tool).

usage: python tools/ncu_lines.py <sass csv from `ncu -i X --page source --csv
       --print-source sass`> <nvdisasm -g listing of the same cubin>
Prints stall-sample shares per role (softmax / MMA issuer / TMA producer /
other) with their top stall reasons, then the top source lines.
"""
import csv
import re
import sys

KERNEL = "paper_2603_10353_b200/csrc/kernels/fa_sm100.cu"


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[1]
    data = rows[2:]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_a = h.index("Address")
    stall = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    base = min(int(r[i_a], 16) for r in data)
    a2l, cur, infunc = {}, None, False
    for line in open(sys.argv[2]):
        s = line.strip()
        if s.startswith(".text"):
            infunc = "fa_sparse_kernel" in s
        if not infunc:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', line)
        if m:
            # inlined helpers: attribute to the call site in the kernel file
            inl = re.search(r'inlined at "([^"]+)", line (\d+)', m.group(3))
            if m.group(1).endswith("fa_sm100.cu"):
                cur = int(m.group(2))
            elif inl and inl.group(1).endswith("fa_sm100.cu"):
                cur = int(inl.group(2))
        m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m:
            a2l[int(m.group(1), 16)] = cur
    src = open(KERNEL).read().split("\n")
    # role by the enclosing branch: find line numbers of role markers
    mark = {k: next(i + 1 for i, l in enumerate(src) if k in l)
            for k in ["TMA producer", "MMA issuer", "softmax warpgroups", "epilogue"]}

    def role(ln):
        if ln is None:
            return "?"
        if mark["TMA producer"] <= ln < mark["MMA issuer"]:
            return "producer"
        if mark["MMA issuer"] <= ln < mark["softmax warpgroups"]:
            return "mma"
        if mark["softmax warpgroups"] <= ln < mark["epilogue"]:
            return "softmax"
        if ln >= mark["epilogue"]:
            return "epilogue/exit"
        return "prologue/helpers"

    tot, by_line = {}, {}
    for r in data:
        ln = a2l.get(int(r[i_a], 16) - base)
        ro = role(ln)
        d = tot.setdefault(ro, {})
        for i in stall:
            d[h[i]] = d.get(h[i], 0) + float(r[i] or 0)
        by_line[ln] = by_line.get(ln, 0) + float(r[i_s] or 0)
    grand = sum(sum(d.values()) for d in tot.values())
    for ro, d in sorted(tot.items(), key=lambda x: -sum(x[1].values())):
        t = sum(d.values())
        top = sorted(d.items(), key=lambda x: -x[1])[:5]
        print(f"{ro:18s} {100 * t / grand:5.1f}%  " + ", ".join(f"{k[6:]} {100 * v / t:.0f}%" for k, v in top))
    print()
    for ln, v in sorted(by_line.items(), key=lambda x: -x[1])[:25]:
        text = src[ln - 1].strip()[:80] if ln else ""
        print(f"{100 * v / grand:5.1f}% L{ln} [{role(ln)}] {text}")


if __name__ == "__main__":
    main()
