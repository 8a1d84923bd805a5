set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp tools/micro/store_pattern.cu && /tmp/sp && /tmp/sp r
for p in 0 1 2 3; do PPLL_GEMM_PROBE=$p python tools/gemm_one.py 8320 384 1536 fwdgelu 20; done
PPLL_GEMM_TMA_STORE=0 python tools/gemm_one.py 8320 384 1536 fwdgelu 20
python tools/gemm_one.py 8320 384 1152 fwd 20
python tools/gemm_one.py 8320 1536 384 dgradmul 20
python tools/gemm_one.py 8320 384 1536 dgrad 20
python tools/gemm_one.py 8192 8192 8192 fwd 5
