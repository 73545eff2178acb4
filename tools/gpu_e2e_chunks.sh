mkdir -p gpurun_out
for n in 1 2 4 8 12 24; do
  XC_HOST_CHUNKS=$n timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 6 --no-cpu-baseline > gpurun_out/e.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/e.json'));print('chunks $n e2e %.0f/s ms %.2f'%(d['e2e']['value'],d['e2e']['ms_per_step']))"
done
nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.width.current --format=csv
