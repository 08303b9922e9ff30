set -x
python tools/emulated_scaling.py c4 --exchange full > gpurun_out/g5_emul_full.txt 2>&1
python tools/emulated_scaling.py c4 --exchange p2p > gpurun_out/g5_emul_p2p.txt 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/g5_pytest.log 2>&1
