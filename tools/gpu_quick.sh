cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest ${PYTESTS:-tests} -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/${TAG:-q}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG:-q}_pytest.log
timeout 600 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/${TAG:-q}_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-q}_launches.csv python bench.py --no-cpu --no-parity --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG:-q}_launches.csv > gpurun_out/${TAG:-q}_launch_summary.txt 2>&1
