"""Map ncu per-instruction warp-stall samples (--page source --print-source sass
--csv) to source lines of the kernel's outermost caller, using nvdisasm -gi of
the same cubin.

    python tools/ncu_stall_map.py stalls.csv disasm.txt <function-substring> [top]
"""
import collections
import csv
import re
import sys


def main():
    csv_path, dis_path, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ia, iss, ins = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Warp Stall Sampling (Not-issued Samples)")
    data = [r for r in rows[2:] if r and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    cur, loc, off2loc = None, None, {}
    for line in open(dis_path):
        m = re.match(r"\s*\.text\.(\S+):", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', line)
        if m:
            loc = (m.group(3) or m.group(1)).split("/")[-1] + ":" + (m.group(4) or m.group(2))
            inner = m.group(1).split("/")[-1] + ":" + m.group(2)
            loc = (loc, inner)
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", line)
        if cur and fn in cur and m:
            off2loc[int(m.group(1), 16)] = loc
    agg, agg_ni = collections.Counter(), collections.Counter()
    tot = 0
    for r in data:
        off = int(r[ia], 16) - base
        s, ns = int(r[iss]), int(r[ins])
        tot += s
        loc = off2loc.get(off, ("?", "?"))
        agg[loc] += s
        agg_ni[loc] += ns
    print("total samples", tot)
    for k, v in agg.most_common(top):
        print(f"{v:8d} {100 * v / tot:5.1f}%  not-issued {agg_ni[k]:8d}  {k[0]:28s} <- {k[1]}")


if __name__ == "__main__":
    main()
