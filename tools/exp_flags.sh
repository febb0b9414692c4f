cd "${GRAFT_REPO_ROOT:-.}"
for f in 0 2; do for c in fibbatch sortbatch buildsum22; do timeout 300 python tools/sweep_timeline.py $c --debug-flags $f | python -c "
import json,sys; d=json.load(sys.stdin); print('flags$f', d['name'], round(d['kernel_ms'],2))"; done; done
