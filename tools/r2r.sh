cat > /tmp/b_hd.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import _lib, ops
from paper_2511_10442_b200.datasets import config_dataset
c, off, k = config_dataset("B"); n, d = c.shape
nb = fg.compute_n_bins(int(np.diff(off).max()), k, d)
ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d, nb)
for i in range(3):
    ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, None, None, False, False)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:k_hd_search -s 1 -c 1 -o gpurun_out/B_hd2 python /tmp/b_hd.py > gpurun_out/B_hd2.log 2>&1
ncu -i gpurun_out/B_hd2.ncu-rep --page source --csv --print-source sass > gpurun_out/B_hd2.sass.csv 2>&1
ncu -i gpurun_out/B_hd2.ncu-rep --page details --csv > gpurun_out/B_hd2.details.csv 2>&1
grep -E '"(Duration|Executed Ipc Active|Issue Slots Busy|Achieved Occupancy|Theoretical Occupancy|Warp Cycles Per Issued Instruction|L1/TEX Hit Rate|L2 Hit Rate|Registers Per Thread)"' gpurun_out/B_hd2.details.csv | awk -F'","' '{print $(NF-2)" | "$NF}'
ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/b_hd.py 2>/dev/null | grep -E "k_hd|k_cell|k_dense|k_tile|k_knn|k_scan" | awk -F'","' '{print $5" "$NF}' | cut -c1-100 | tail -12
