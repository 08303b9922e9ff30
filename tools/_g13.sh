python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "sharded or p2p or delta" > gpurun_out/g13_pytest.log 2>&1
python -m pytest tests/test_flavours.py -q -p no:cacheprovider > gpurun_out/g13_flavours.log 2>&1
python tools/emulated_scaling.py c4 --exchange p2p > gpurun_out/g13_emul_p2p.txt 2>&1
