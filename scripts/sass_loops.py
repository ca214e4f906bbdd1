"""Find the hot epilogue loops of k_sweep_tc in a cuobjdump -sass dump: for
each LDTM (tcgen05.ld), the smallest backward branch enclosing it; print the
loop body size and a few opcode counts.  python scripts/sass_loops.py dump.sass [filter]"""
import re
import sys
from collections import Counter

txt = open(sys.argv[1]).read()
filt = sys.argv[2] if len(sys.argv) > 2 else "ILi16ELb1E"
for f in re.split(r'\n\s*Function : ', txt)[1:]:
    name = f.split('\n')[0]
    if filt not in name:
        continue
    ins = []
    for l in f.split('\n'):
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s*(.*?);', l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = [a for a, _ in ins]
    print(name[-50:], len(ins))
    for k, (a, t) in enumerate(ins):
        if 'LDTM' not in t:
            continue
        best = None
        for j in range(k, len(ins)):
            m = re.search(r'BRA (?:`\()?(?:\.L_x_\d+)?0x([0-9a-f]+)', ins[j][1])
            if m and 'BRA' in ins[j][1]:
                tgt = int(m.group(1), 16)
                if tgt <= a:
                    best = (tgt, ins[j][0])
                    break
        if not best:
            continue
        body = [t for a2, t in ins if best[0] <= a2 <= best[1]]
        ops = Counter(re.sub(r'^@!?U?P\w+\s+', '', t).split()[0] for t in body)
        print(f"  loop {best[0]:#x}-{best[1]:#x}: {len(body)} instr  "
              + " ".join(f"{o}={ops[o]}" for o in ('DADD', 'VOTE.ALL', 'VOTE.ANY', 'LDS.128', 'LDS.64', 'LDL', 'STL', 'SHFL.BFLY', 'STG.E.NA.64')
                         if ops[o]))
