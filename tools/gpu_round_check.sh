set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f1_smi.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/f1_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/f1_bench.json 2> gpurun_out/f1_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f1_ref.json 2> gpurun_out/f1_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f1_launches.csv python bench.py --no-cpu-baseline --no-e2e > gpurun_out/f1_ncu.log 2>&1
echo done
