# ncu --set full of the GEMM kernels at chosen ratios (tag $1)
TAG=${1:-x}
set -x
for r in 0.9 0.25; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_q2 -s 3 -c 1 -o gpurun_out/gq_${TAG}_$r -f python tools/gemm_time.py --ops q --ratios $r --orders 0 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_o_kernel -s 5 -c 1 -o gpurun_out/godisp_${TAG}_$r -f python tools/gemm_time.py --ops disp --ratios $r --orders 0 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_o_update -s 5 -c 1 -o gpurun_out/goupd_${TAG}_$r -f python tools/gemm_time.py --ops upd --ratios $r --orders 0 > /dev/null 2>&1
done
ls gpurun_out | grep $TAG
