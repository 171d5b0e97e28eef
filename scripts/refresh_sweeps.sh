set -e
O=gpurun_out/sweeps; mkdir -p $O
python -m paper_1506_08503_b200.sweep --kind count --out $O/sweep_count_cuda.csv
python -m paper_1506_08503_b200.sweep --kind count --device-resident --counts 1024,16384,65536,262144,1048576,4194304,16777216,67108864,268435456,1073741824 --out $O/sweep_count_cuda_device.csv
python -m paper_1506_08503_b200.sweep --kind length --n-messages 100000 --lengths 16,64,256,1024,4096 --out $O/sweep_length_cuda.csv
python -m paper_1506_08503_b200.sweep --kind length --device-resident --n-messages 262144 --lengths 16,32,64,256,1024,4096 --out $O/sweep_length_cuda_device.csv
wc -l $O/*.csv
