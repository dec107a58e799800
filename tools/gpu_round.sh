#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench (+ reference arm), ncu launch list of the bench
# command, and (FULL=1) an ncu --set full capture of one steady update round's pair-phase
# kernels (round 21 of a T1=2 T2=15 C2-shape schedule).  Outputs under gpurun_out/<tag>_*.
cd "$(dirname "$0")/.."
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
if [ "${REF:-1}" = 1 ]; then
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/${TAG}_bench_ref.log 2>&1
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --no-cpu --no-parity --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1
if [ "${FULL:-0}" = 1 ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${REGEX:-tc3_pairs|tc_stage|decide}" -s ${SKIP:-139} -c ${CNT:-8} \
   -o gpurun_out/${TAG}_round_full -f python tools/prof_rounds.py 1000000 128 2 15 > gpurun_out/${TAG}_ncu_full.log 2>&1
python tools/ncu_to_json.py gpurun_out/${TAG}_round_full.ncu-rep gpurun_out/${TAG}_pair_phase_ncu.json \
   "ncu --set full --clock-control none -k regex:${REGEX:-tc3_pairs|tc_stage|decide} -s ${SKIP:-139} -c ${CNT:-8}, tools/prof_rounds.py 1000000 128 2 15 (update round 21)" \
   > gpurun_out/${TAG}_ncu_json.log 2>&1
fi
echo done
