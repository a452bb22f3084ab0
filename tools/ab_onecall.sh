# A/B: one-call multiply (C allocated at nnz(M) up front, compaction queued behind the scan) vs begin/end on cfg2
for v in 22 30 22 30; do python -c "
import sys, runpy, json, io, contextlib
sys.path.insert(0,'.')
import paper_2111_09947_b200.multiply as m
m.ONE_CALL_MAX_NNZ = 1 << $v
sys.argv=['bench.py','--no-cpu-baseline','--steps','20']
buf=io.StringIO()
try:
    with contextlib.redirect_stdout(buf):
        runpy.run_path('bench.py', run_name='__main__')
except SystemExit:
    pass
d=json.loads(buf.getvalue().strip().splitlines()[-1])
print($v, round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['phase_ms'].items()}, round(d['e2e']['ms_per_step'],3))
" 2>&1 | tail -2; done
