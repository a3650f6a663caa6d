"""Attribute an ncu SASS source-page export (tools/ncu_export.sh *_source.csv.gz) to CUDA source
lines using the line table of the local build (nvdisasm -gi on the object's cubin; -lineinfo).
Run here (no GPU):  python tools/sass_lines.py <obj.o> <source.csv.gz> <function-substring> [N]
Prints the top source lines (innermost inline frame, and the outermost frame inside the
function's own file) by warp-stall samples, with executed instructions."""
import collections, csv, gzip, os, re, subprocess, sys, tempfile


def line_table(obj):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    tab = {}
    fn, frames, pending = None, [], []
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1); frames = []; pending = []; tab[fn] = {}
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
        if m:
            pending.append((os.path.basename(m.group(1)), int(m.group(2))))
            if m.group(3):
                pending.append((os.path.basename(m.group(3)), int(m.group(4))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and fn:
            if pending:
                frames, pending = pending, []
            tab[fn][int(m.group(1), 16)] = list(frames)
    return tab


def main(obj, csvgz, sub, n=40):
    tab = line_table(obj)
    rows = list(csv.reader(gzip.open(csvgz, "rt")))
    fn, hdr, data = None, None, collections.defaultdict(list)
    for r in rows:
        if not r:
            continue
        if r[0] == "Kernel Name":
            fn = r[1]; continue
        if r[0] == "Address":
            hdr = r; continue
        data[fn].append(dict(zip(hdr, r)))
    for f, L in data.items():
        if sub not in f:
            continue
        # the mangled name: match by the instruction count of the cubin function
        cands = [k for k, v in tab.items() if len(v) == len(L)]
        if not cands:
            print("no line table match for", f); continue
        t = tab[cands[0]]
        base = int(L[0]["Address"], 16)
        agg = collections.defaultdict(lambda: [0, 0])
        tot = 0
        for d in L:
            off = int(d["Address"], 16) - base
            s = int(d["Warp Stall Sampling (All Samples)"] or 0)
            i = int(d["Instructions Executed"] or 0)
            fr = t.get(off) or [("?", 0)]
            key = f"{fr[0][0]}:{fr[0][1]}" + (f" <- {fr[-1][0]}:{fr[-1][1]}" if len(fr) > 1 else "")
            agg[key][0] += s; agg[key][1] += i; tot += s
        print(f"== {f[:100]}  ({tot} samples)")
        for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(n)]:
            print(f"  {100*s/tot:5.1f}%  {i:>11d}  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
