# Round-2 final set on one 4-GPU box: the 1-GPU lines on GPU 0, then the multi-GPU set.
set -x
O=gpurun_out/fin1b; mkdir -p $O
export CUDA_VISIBLE_DEVICES=0
B="timeout 300 python bench.py"
$B > $O/b1.json 2>>$O/err.log
$B --seq-len 131072 > $O/b1_131k.json 2>>$O/err.log
$B --workload cfg1 --steps 30 > $O/b1_cfg1.json 2>>$O/err.log
$B --workload cfg2 --steps 20 > $O/b1_cfg2.json 2>>$O/err.log
$B --workload cfg4 --steps 20 > $O/b1_cfg4.json 2>>$O/err.log
$B --dynamic > $O/b1_dyn.json 2>>$O/err.log
$B --seq-len 131072 --dynamic > $O/b1_131k_dyn.json 2>>$O/err.log
$B --impl reference --steps 3 --warmup 1 > $O/ref1.json 2>>$O/err.log
(timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? >> $O/smoke.log)
unset CUDA_VISIBLE_DEVICES
sed -i 's#O=gpurun_out/fin4;#O=gpurun_out/fin4b;#' scripts/gpurun_final_4gpu.sh
bash scripts/gpurun_final_4gpu.sh
