set -x
TAG=${TAG:-r02_v8}
mkdir -p gpurun_out
python -c "import bench; print(bench.source_hash())" > gpurun_out/${TAG}_srchash.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -4 > gpurun_out/${TAG}_pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/${TAG}_bench.json
timeout 300 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/${TAG}_bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ddl_chain -s 3 -c 1 -f -o gpurun_out/${TAG}_step python scripts/profile_step.py --warmup 3 > gpurun_out/${TAG}_step.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_reduce -s 3 -c 1 -f -o gpurun_out/${TAG}_k5 python scripts/profile_k5.py --warmup 3 > gpurun_out/${TAG}_k5.log 2>&1
cat gpurun_out/${TAG}_pytest_gpu.txt gpurun_out/${TAG}_smoke.txt
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['local_reduce'])"
cat gpurun_out/${TAG}_bench_reference.json
ls -la gpurun_out
ncu -i gpurun_out/${TAG}_step.ncu-rep --page details --csv > gpurun_out/${TAG}_step_details.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_k5.ncu-rep --page details --csv > gpurun_out/${TAG}_k5_details.csv 2>/dev/null
# keep gpurun_out under gpurun's 64 MiB copy-back limit: the K5 report's details are extracted above
rm -f gpurun_out/${TAG}_k5.ncu-rep
du -sh gpurun_out
