#!/bin/bash
# evidence for the fp16-split state: ncu launch list + full capture of one VGG step (reports kept
# on the box in /tmp, summaries in gpurun_out), the per-layer report of every config, the method table
tag=${1:-ev}; out=gpurun_out/$tag; mkdir -p $out; R=/tmp/ncu_$tag; mkdir -p $R
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches.csv $B > $out/ncu_launch.log 2>&1
echo "launch list rc=$?"
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -s 12 -c 12 -o $R/step $B1 > $out/ncu_full.log 2>&1
echo "full rc=$?"
python tools/make_traffic.py $R/step.ncu-rep vgg16 $out/ncu_step_summary.json auto > $out/traffic.log 2>&1; echo "traffic rc=$?"
cp profiles/ncu_traffic_vgg16.json $out/ 2>/dev/null
ncu --set full --clock-control none -k regex:split_spec_kernel -s 13 -c 1 -o $R/prepass $B1 > $out/ncu_prepass.log 2>&1; echo "prepass rc=$?"
python -c "import sys,json; sys.path.insert(0,'tools'); from ncu_summary import summarize; print(json.dumps(summarize('$R/prepass.ncu-rep'), indent=1))" > $out/ncu_prepass_summary.json 2>&1
ncu --set full --clock-control none -k regex:direct -s 1 -c 1 -o $R/direct $B1 > $out/ncu_direct.log 2>&1; echo "direct rc=$?"
python -c "import sys,json; sys.path.insert(0,'tools'); from ncu_summary import summarize; print(json.dumps(summarize('$R/direct.ncu-rep'), indent=1))" > $out/ncu_direct_summary.json 2>&1
timeout 2400 python tools/report.py > $out/report.json 2> $out/report.err; echo "report rc=$?"
timeout 1500 python tools/method_table.py > $out/method_table.json 2> $out/method_table.err; echo "table rc=$?"
du -sh $out
