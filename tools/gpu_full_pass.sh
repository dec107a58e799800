#!/bin/bash
# One complete GPU-box pass for the round's evidence (outputs gpurun_out/${TAG}_*):
#   gpu tests + smoke; C2 bench (+ the reference arm); the bench's ncu launch list and the
#   per-round table; one ncu --set full capture of a steady round's pair phase (round 21,
#   tc3 + stage + decide) -> <tag>_pair_phase_ncu.json; bench lines for C1, C2c, C3, C4;
#   (sanitizers: tools/sanitize.sh, run separately where compute-sanitizer is allowed).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-full}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_c2_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_c2_bench.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/${TAG}_c2_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --no-cpu --no-parity --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_c2_launch_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_rounds.csv \
   python tools/prof_rounds.py 1000000 128 4 15 > /dev/null 2>&1
python tools/round_table.py gpurun_out/${TAG}_rounds.csv > gpurun_out/${TAG}_c2_rounds.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc3_pairs|tc_stage|decide" -s 139 -c 8 \
   -o gpurun_out/${TAG}_round_full -f python tools/prof_rounds.py 1000000 128 2 15 > gpurun_out/${TAG}_ncu_full.log 2>&1
python tools/ncu_to_json.py gpurun_out/${TAG}_round_full.ncu-rep gpurun_out/${TAG}_pair_phase_ncu.json \
   "ncu --set full --clock-control none -k regex:tc3_pairs|tc_stage|decide -s 139 -c 8, tools/prof_rounds.py 1000000 128 2 15 (update round 21)" \
   > gpurun_out/${TAG}_ncu_json.log 2>&1
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/${TAG}_c1_bench.log 2>&1
timeout 900 python bench.py --config c2c --no-cpu --steps 3 --warmup 3 > gpurun_out/${TAG}_c2c_bench.log 2>&1
timeout 1200 python bench.py --config c3 --no-cpu --steps 2 --warmup 3 > gpurun_out/${TAG}_c3_bench.log 2>&1
timeout 1500 python bench.py --config c4 --no-cpu --steps 2 --warmup 3 > gpurun_out/${TAG}_c4_bench.log 2>&1
# (compute-sanitizer passes: tools/sanitize.sh -- closed on this pool since r2cj; last results profiles/r2bp_sanitizers.txt)
echo done
