#!/bin/bash
# What the driver runs at round end: GPU suite, smoke(), both bench arms (default flags)
# usage (gpurun): bash tools/gpu_driver_check.sh <tag>
out=gpurun_out/${1:-driver}; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rf > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 900 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err; echo "ref rc=$?"
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench rc=$?"
tail -c 600 $out/bench_default.json
