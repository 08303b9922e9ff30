set -x
python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_parity.py::test_c4_end_to_end_10_sweeps --deselect tests/test_gpu_parity.py::test_c4_flip_census_sweeps_1_to_3 > gpurun_out/g3_pytest.log 2>&1
python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
python -m pytest tests/test_gpu_parity.py -k "c4_end_to_end" -q -s -p no:cacheprovider > gpurun_out/g3_c4e2e.log 2>&1
python tools/flip_census_oracle.py --config c4 --sweeps 10 --out gpurun_out/g3_rcensus.jsonl > gpurun_out/g3_rcensus.log 2>&1
python tools/prof_run.py --config c4 --sweeps 2 > gpurun_out/g3_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_sacd_rows_mma_gram|k_mttkrp_lean_dyn" -s 7 -c 6 -o gpurun_out/g3_prof python tools/prof_run.py --config c4 --sweeps 2 > gpurun_out/g3_ncu.log 2>&1
