set -x
SACD_LIB=libsacd_tuning.so python tools/mttkrp_tune.py --config c4 --variants 0,50,51,52,53,54,55,56,57 --sweeps 6 > gpurun_out/g2_tune.txt 2>&1
python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
python tools/flip_census.py --config c4 --sweeps 10 --out gpurun_out/g2_census.jsonl > gpurun_out/g2_census.log 2>&1
python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_parity.py::test_c4_end_to_end_10_sweeps > gpurun_out/g2_pytest.log 2>&1
