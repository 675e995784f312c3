# NVTX ranges: ncu filtered to one C-ABI entry point's kernels
mkdir -p gpurun_out
ncu --nvtx --nvtx-include "fo_gemm_qkv/" --metrics gpu__time_duration.sum --csv -c 5 \
  python tools/gemm_time.py --ops qkv --orders 0 --ratios 0.25 --eager > gpurun_out/nvtx_qkv.csv 2>&1
grep -c "gemm_q2_kernel" gpurun_out/nvtx_qkv.csv; grep -v "^==" gpurun_out/nvtx_qkv.csv | cut -c1-200 | head -8
