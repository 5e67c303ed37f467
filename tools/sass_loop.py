"""Instruction count of the SpMV's interior pair loop (the loop whose body has 16 unpredicated FHFMAs)
and of the whole kernel, from `cuobjdump -sass` text: python tools/sass_loop.py FILE.sass"""
import re
import sys

lines = [l for l in open(sys.argv[1]) if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, t) in enumerate(ins):
    m = re.match(r"(@!?U?P\d\s+)?BRA(\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
    if not m:
        continue
    tgt = int(m.group(3), 16)
    if tgt >= a or tgt not in addr:
        continue
    body = ins[addr[tgt]:i + 1]
    n_fh = sum(1 for _, x in body if x.startswith("FHFMA"))
    if n_fh == 16 and (best is None or len(body) < len(best)):
        best = body
print("kernel instructions:", len(ins))
if best:
    print("interior loop instructions:", len(best))
    from collections import Counter
    c = Counter(x.split()[0] if not x.startswith("@") else x.split()[1] for _, x in best)
    print(" ".join(f"{k}:{v}" for k, v in c.most_common()))
