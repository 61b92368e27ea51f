timeout 300 python tools/e2e_prof.py B 6 > gpurun_out/e2e_B2.txt 2>&1
head -6 gpurun_out/e2e_B2.txt
timeout 300 python tools/e2e_prof.py C 2 2>&1 | head -5
