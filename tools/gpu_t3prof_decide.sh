cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
GRNND_B200_LIB=paper_2510_02774_b200/_build/variants/t3prof/libgrnnd_b200.so timeout 600 python tools/t3prof.py > gpurun_out/r2cf_t3prof.txt 2>&1
for spec in "decide:15:r16" "decide:2:r3"; do
  IFS=: read k s r <<< "$spec"
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 \
     -o gpurun_out/r2cf_${k}_${r} -f python tools/prof_rounds.py 1000000 128 2 15 > gpurun_out/r2cf_${k}_${r}.log 2>&1
  ncu -i gpurun_out/r2cf_${k}_${r}.ncu-rep --page source --csv --print-source sass > gpurun_out/r2cf_${k}_${r}_sass.csv 2>/dev/null
done
