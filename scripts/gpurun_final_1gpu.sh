set -x
O=gpurun_out/fin1; mkdir -p $O
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
(timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/pytest.log)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3_p1.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
TD_CALIBRATE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine_split" --launch-skip 2 -c 2 -o $O/ncu_cfg3_131k python bench.py --seq-len 131072 --steps 2 --warmup 3 > $O/ncu_131k.log 2>&1
TD_CALIBRATE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine_split" --launch-skip 2 -c 2 -o $O/ncu_cfg3_1m python bench.py --steps 2 --warmup 3 > $O/ncu_1m.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_f32|k2_combine_split" --launch-skip 2 -c 2 -o $O/ncu_cfg1 python bench.py --workload cfg1 --steps 2 --warmup 3 > $O/ncu_cfg1.log 2>&1
ls -la $O
