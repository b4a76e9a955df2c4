#!/bin/bash
# Round-2 GPU session: build, the multicast probe, the GPU tests, smoke, bench lines.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- bash tools/gpu_r02.sh TAG [extra bench args]
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 300 python tools/probe_multicast.py > $O/probe.json 2> $O/probe.err; echo "probe rc=$? $(cat $O/probe.json)"
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "gputest rc=$? $(tail -1 $O/gputest.log)"
grep -E "FAILED|Error" $O/gputest.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)"
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench3.json 2> $O/bench3.err; echo "bench3 rc=$?"; tail -c 1500 $O/bench3.json
timeout 600 python bench.py --workload config4 --steps 10 --warmup 3 --skip-cpu --e2e-steps 2 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"; tail -c 800 $O/bench4.json
