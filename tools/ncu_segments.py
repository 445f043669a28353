"""Group SASS instructions of an ncu report into runs of equal execution count
(= basic blocks) and print the heaviest ones with their opcode mix."""
import collections, csv, io, re, subprocess, sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
E = "Instructions Executed"
cnt = [float(r[ix[E]] or 0) for r in data]
segs, start = [], 0
for i in range(1, len(data) + 1):
    if i == len(data) or abs(cnt[i] - cnt[start]) > 0.5:
        segs.append((start, i - 1, cnt[start]))
        start = i
tot = sum(cnt)
for a, b, c in sorted(sorted(segs, key=lambda s: -(s[1] - s[0] + 1) * s[2])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]):
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", data[k][ix["Source"]].strip()).split(" ")[0].split(".")[0]
                              for k in range(a, b + 1))
    print(f"[{a:5d}-{b:5d}] n={b - a + 1:4d} exec={c:.3e} share={(b - a + 1) * c / tot * 100:5.1f}%  {dict(ops.most_common(6))}")
