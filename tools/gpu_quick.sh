#!/bin/bash
# quick GPU check: build, gpu tests (optional), bench with/without an env toggle, kprof
TAG=${1:-q}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail -30 gpurun_out/${TAG}_build.log; exit 1; }
for w in "$@"; do case $w in
tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 ;;
bench) timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench.json'));print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'roof',d['roofline']['frac'],d['clocks'])" ;;
bench_pdl) RN_PDL=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_pdl.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench_pdl.json'));print('PDL value',d['value'],'ms',d['ms_per_step'])" ;;
kprof) KPROF_NOSIDE=1 RN_PDL=0 KPROF_NOGRAPH=1 timeout 300 python tools/kprof.py 5 8 gpurun_out/${TAG}_kprof.txt 2>&1 | grep -v Warn | head -60 ;;
esac; done
