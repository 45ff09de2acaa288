mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ll.py -q -m gpu --timeout 600 2>&1 | tail -3 > gpurun_out/r02_v2_ll.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_v2_smoke.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_v2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_v2_smoke_ncu.txt 2>&1; echo "ncu_rc=$?" >> gpurun_out/r02_v2_smoke_ncu.txt
DDL_BENCH_SAME_GPU=1 OUT=gpurun_out/decisions_dry timeout 1200 bash scripts/nvlink_decisions.sh 2 > gpurun_out/r02_v2_decisions_dry.log 2>&1
timeout 900 python scripts/train_ddp.py --table1 --gpus 1 --model resnet50 --steps 10 > gpurun_out/r02_v2_table1_resnet50.txt 2>&1
timeout 900 python scripts/train_ddp.py --table1 --gpus 1 --model unet3d --steps 10 > gpurun_out/r02_v2_table1_unet3d.txt 2>&1
cat gpurun_out/r02_v2_ll.txt gpurun_out/r02_v2_smoke.txt gpurun_out/r02_v2_smoke_ncu.txt; tail -5 gpurun_out/r02_v2_decisions_dry.log; cat gpurun_out/r02_v2_table1_*.txt
