python tools/oracle_breakdown.py c4 > gpurun_out/g11_oracle_breakdown.txt 2>&1
