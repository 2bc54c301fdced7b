#!/bin/bash
# Full evidence pass on the GPU box: GPU tests, bench (both arms), ncu launch list + full captures,
# summaries under profiles/ (copied back through gpurun_out/profiles/).
# usage: tools/round_gpu.sh <tag>
TAG=${1:-r1}
mkdir -p gpurun_out/profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 400 gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; tail -c 300 gpurun_out/${TAG}_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
python tools/ncu_summary.py launches gpurun_out/${TAG}_launches.csv gpurun_out/profiles/${TAG}_launches.txt > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma -c 4 -o gpurun_out/${TAG}_umma python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${TAG}_ncu_umma.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'head|cut|adam|stats|dz1' -c 7 -o gpurun_out/${TAG}_misc python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${TAG}_ncu_misc.log 2>&1
python tools/ncu_summary.py report gpurun_out/${TAG}_umma.ncu-rep gpurun_out/profiles/${TAG}_umma_full.txt > /dev/null
python tools/ncu_summary.py report gpurun_out/${TAG}_misc.ncu-rep gpurun_out/profiles/${TAG}_misc_full.txt > /dev/null
python tools/traffic_json.py gpurun_out/profiles/traffic.json gpurun_out/${TAG}_umma.ncu-rep gpurun_out/${TAG}_misc.ncu-rep > /dev/null
# SR (natural gradient) step: launch list of one solve and the step rate at N = 10k
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_sr_launches.csv python scripts/sr_rate.py 10000 0 > gpurun_out/${TAG}_sr_ncu.log 2>&1
python tools/ncu_summary.py launches gpurun_out/${TAG}_sr_launches.csv gpurun_out/profiles/${TAG}_sr_launches.txt > /dev/null
timeout 300 python scripts/sr_rate.py 10000 3 > gpurun_out/profiles/${TAG}_sr_rate.txt 2>&1
cp gpurun_out/${TAG}_bench.json gpurun_out/profiles/${TAG}_bench.json; cp gpurun_out/${TAG}_bench_ref.json gpurun_out/profiles/${TAG}_bench_ref.json
head -24 gpurun_out/profiles/${TAG}_launches.txt
ls gpurun_out/profiles
