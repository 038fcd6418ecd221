#!/bin/bash
# One gpurun round trip: GPU parity tests, a short bench, launch lists.
# usage: tools/gpu_check.sh TAG [pytest-args]
TAG=${1:-x}; shift
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/pytest_$TAG.log 2>&1; tail -4 gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('matvec/s', round(d['value'],2), 'ms', round(d['ms_per_step'],3), 'gather GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), 'tts', d['time_to_solution'])" || tail -5 gpurun_out/bench_$TAG.err
for w in matvec refresh; do
  timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${w}_$TAG.csv python tools/profile_step.py --what $w > /dev/null 2>&1
done
python tools/launches.py gpurun_out/launches_matvec_$TAG.csv gpurun_out/launches_refresh_$TAG.csv 2>&1 | cut -c1-120
