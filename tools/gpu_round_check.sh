# Round-end evidence on one B200: gpu tests, smoke, bench line (with cpu baseline + e2e),
# reference arm, ncu launch list of the bench command, ncu --set full of sweep 2's kernels
# (MTTKRP, row update, Gram of each mode; c4), every config's bench line.
# Usage: bash tools/gpu_round_check.sh TAG
T=${1:-f}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --no-cpu-baseline --no-e2e --reps 1 > gpurun_out/${T}_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mttkrp|k_sacd_rows|k_gram_stream" --launch-skip 9 -c 9 -o gpurun_out/${T}_full python tools/prof_run.py --sweeps 2 > gpurun_out/${T}_full.log 2>&1
bash tools/bench_all.sh gpurun_out/${T}_bench_all.jsonl
echo done
