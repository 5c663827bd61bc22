#!/bin/bash
# fp16 split round 2: the new range tests + GPU suite, then the ncu launch list of the default bench
out=gpurun_out/${1:-f16c}; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "f16_split or operand_split or padded_row or delta" > $out/pytest_new.log 2>&1; echo "rc=$?" >> $out/pytest_new.log
tail -3 $out/pytest_new.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $out/ncu.log 2>&1; echo "ncu rc=$?"
