# Round-end evidence on one B200: gpu tests, smoke, bench line (with cpu baseline + e2e),
# reference arm, ncu launch list of the bench command, ncu --set full of the three MTTKRP
# launches of sweep 7 (c4).  Usage: bash tools/gpu_round_check.sh TAG
T=${1:-f}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mttkrp --launch-skip 19 -c 3 -o /tmp/${T}_mttkrp python tools/prof_run.py --sweeps 7 > gpurun_out/${T}_full.log 2>&1
ncu -i /tmp/${T}_mttkrp.ncu-rep --page raw --csv > gpurun_out/${T}_mttkrp_full.csv
echo done
