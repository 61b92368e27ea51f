# compile one csrc file for sm_100a and list registers / spills per kernel:
#   bash tools/ptxas_check.sh fg_grad.cu [name-filter]
cd "$(dirname "$0")/../paper_2511_10442_b200/csrc" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
     -I../../include -c "$1" -o /tmp/ptxas_check.o 2>&1 | grep -E "error|warning" | grep -v "ptxas info"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
     -I../../include -c "$1" -o /tmp/ptxas_check.o 2>&1 | grep -A2 "${2:-Compiling}" | grep -E "Compiling|registers|spill" |
  sed 's/ptxas info    : //; s/Compiling entry function//; s/for .sm_100a.//' | paste - - - | cut -c1-220
