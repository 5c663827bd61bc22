#!/bin/bash
# fp16 split: GPU suite, smoke, default bench (VGG-16) and the mixed-split bench for A/B
out=gpurun_out/${1:-f16b}; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
CLB_SPLIT=mixed timeout 900 python bench.py --no-cpu-baseline > $out/bench_vgg16_mixed.json 2> /dev/null; echo "mixed rc=$?"
timeout 900 python bench.py --workload alexnet --no-cpu-baseline > $out/bench_alexnet.json 2> /dev/null; echo "alexnet rc=$?"
