#!/bin/bash
OUT=gpurun_out/b12; mkdir -p $OUT
timeout 900 ncu --set full -k regex:"k_cg_(xr|ap|p)$" --launch-skip 3 -c 3 -o $OUT/cgvec python scripts/c5_fit_probe.py 3 > $OUT/cgvec.log 2>&1
timeout 900 ncu --set full -k regex:"k_mr_(a|r|w)$" --launch-skip 3 -c 3 -o $OUT/mrvec python -c "
import sys, os; sys.argv=['x','3']; os.environ['GVT_TEST_SOLVER']='1'
exec(open('scripts/c5_fit_probe.py').read().replace('ctx.set_option(G.OPT_GRAPHS, 0)', 'ctx.set_option(G.OPT_GRAPHS, 0); ctx.set_option(G.OPT_SOLVER, 1)'))
" > $OUT/mrvec.log 2>&1
ls -la $OUT
