for v in default norev; do
  if [ $v = default ]; then lib=""; else lib=paper_2510_02774_b200/_build/variants/$v/libgrnnd_b200.so; fi
  GRNND_B200_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lt_$v.csv python tools/prof_rounds.py 1000000 128 2 15 > /dev/null 2>&1
done
