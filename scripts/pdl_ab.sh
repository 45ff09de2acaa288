timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ll.py -q -x 2>&1 | tail -2
S=1024,65536,524288,1048576,8196000,31502336
for pdl in 1 0; do
  DDL_PDL=$pdl python scripts/lb_microbench.py --graph --sizes $S --dims 8 | sed "s/^/pdl$pdl,graph,/"
  DDL_PDL=$pdl python scripts/lb_microbench.py --sizes $S | sed "s/^/pdl$pdl,eager,/"
  DDL_PDL=$pdl python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('pdl$pdl bench', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_step'], d['config']['bucket_us'], d['local_reduce']['achieved'])"
done
