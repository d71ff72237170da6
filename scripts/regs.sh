#!/bin/bash
# register / stack usage of the CTA-pair GEMM instantiations in libgvt.so
cuobjdump -res-usage paper_2009_01054_b200/libgvt.so 2>/dev/null | python3 -c "
import re, sys
f = None
for l in sys.stdin:
    m = re.search(r'Function (\S+):', l)
    if m: f = m.group(1); continue
    if f and 'k_gemm2_x3' in f and 'REG:' in l:
        p = re.search(r'ILi(\d)ELi(\d)', f)
        print('PREC%s EPI%s' % p.groups(), ' '.join(l.split()[:2]))
"
