"""Per-source-line instruction / stall-sample shares of one kernel in an ncu report.

    python tools/ncu_lines.py gpurun_out/rep.ncu-rep <kernel-regex> [launch-index] [top]
    STPC_SORT=stall_long_sb python tools/ncu_lines.py ...   # rank by one stall column
    STPC_FUNC=fit_pair_kernelILb1 python tools/ncu_lines.py ...  # pick a template instantiation

Maps the report's SASS page (addresses) to CUDA source lines through the
line table of the in-tree library's cubins (nvdisasm -g), because the CSV
source page carries no metrics for CUDA lines.  Needs the .so the report was
taken with (built with -lineinfo).
"""

import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("STPC_B200_LIB", os.path.join(ROOT, "paper_2008_06972_b200", "libstpc_b200.so"))
CSRC = os.environ.get("STPC_CSRC", os.path.join(ROOT, "paper_2008_06972_b200", "csrc"))


def line_table(func_regex):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        lines = dis.split("\n")
        starts = [i for i, l in enumerate(lines) if re.match(r"^_ZN4stpc\w*:$", l) and re.search(func_regex, l)]
        if not starts:
            continue
        cur, table = None, {}
        for l in lines[starts[0] + 1:]:
            if l.startswith("//----"):
                break
            m = re.search(r'//## File "(.*)", line (\d+)', l)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
            if m and cur:
                table[int(m.group(1), 16)] = cur
        return table
    return {}


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    # one launch at a time: the source page of a multi-launch report repeats
    # the first launch's counters otherwise
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                          "--launch-skip", str(idx), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Address":
            cur = {"hdr": r, "rows": []}
            blocks.append(cur)
        elif cur is not None and r and r[0].startswith("0x"):
            cur["rows"].append(r)
    blk = blocks[0]
    h, data = blk["hdr"], blk["rows"]
    ie = h.index("Instructions Executed")
    # STPC_SORT=<column> (e.g. stall_long_sb) ranks lines by that sample column
    smp = h.index(os.environ.get("STPC_SORT", "# Samples"))
    # the cubin function whose line table maps the addresses: STPC_FUNC (a
    # regex over mangled names, e.g. fit_pair_kernelILb1 for the <true>
    # instantiation) -- a template kernel's instantiations share a base name,
    # and the first match is not necessarily the profiled one
    fname = os.environ.get("STPC_FUNC") or re.sub(r"[<(].*", "", kre)
    table = line_table(fname)
    base = int(data[0][0], 16)
    agg = collections.defaultdict(lambda: [0, 0])
    for r in data:
        k = table.get(int(r[0], 16) - base, ("?", 0))
        if r[ie].isdigit():
            agg[k][0] += int(r[ie])
        if r[smp].isdigit():
            agg[k][1] += int(r[smp])
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    src = {}
    for f in glob.glob(os.path.join(CSRC, "*.cu*")):
        src[os.path.basename(f)] = open(f).read().split("\n")
    print(f"{kre} #{idx}: {ti} warp instructions, {ts} samples")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1 if "STPC_SORT" in os.environ else 0])[:top]:
        txt = src[k[0]][k[1] - 1].strip()[:80] if k[0] in src and k[1] > 0 else ""
        print(f"{k[0]:>14}:{k[1]:<5} inst {100 * v[0] / ti:5.1f}%  smp {100 * v[1] / ts:5.1f}%  {txt}")


if __name__ == "__main__":
    main()
