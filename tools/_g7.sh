set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g7_smi.txt
python bench.py > gpurun_out/g7_bench.json 2> gpurun_out/g7_bench.err
/usr/bin/time -v python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g7_ref.json 2> gpurun_out/g7_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g7_smoke.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g7_pytest.log 2>&1
python bench.py --no-cpu-baseline --no-e2e --reps 1 > gpurun_out/g7_plain.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g7_launches.csv python bench.py --no-cpu-baseline --no-e2e --reps 1 > gpurun_out/g7_ncu.log 2>&1
