bash tools/ncu_src.sh C_hd C k_hd_search
python tools/ncu_table.py gpurun_out/C_hd.raw.csv 2>&1 | head -60
python tools/sass_hot.py gpurun_out/C_hd.sass.csv 40 2>&1 | head -70
