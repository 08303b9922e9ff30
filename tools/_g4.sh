set -x
python tools/sweep_ab.py --config c4 --variants "default;gram_variant=2" > gpurun_out/g4_ab.txt 2>&1
python tools/emulated_scaling.py c4 --exchange p2p > gpurun_out/g4_emul_p2p.txt 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/g4_pytest.log 2>&1
./tools/gather_bench 67108864 L2_5MB zipf ldg_w32 > gpurun_out/g4_gplain.log 2>&1 && ncu --set full --clock-control none -k regex:"g_ldg|g_bulk" -c 4 -o gpurun_out/g4_gather ./tools/gather_bench 67108864 L2_5MB zipf ldg_w32 > gpurun_out/g4_ncu.log 2>&1
