cd /root/repo
TAG=r1f
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc3_pairs|tc_stage|decide" -s 139 -c 8 \
   -o gpurun_out/${TAG}_round_full -f python tools/prof_rounds.py 1000000 128 2 15 > gpurun_out/${TAG}_ncu_full.log 2>&1
python tools/ncu_to_json.py gpurun_out/${TAG}_round_full.ncu-rep gpurun_out/${TAG}_pair_phase_ncu.json \
   "ncu --set full --clock-control none -k regex:tc3_pairs|tc_stage|decide -s 139 -c 8, tools/prof_rounds.py 1000000 128 2 15 (update round 21)" \
   > gpurun_out/${TAG}_ncu_json.log 2>&1
