mkdir -p gpurun_out/r02e
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p.L2_cache_size if hasattr(p,'L2_cache_size') else '', p)"
nvidia-smi -q | grep -i -A2 "persist" | head
for MB in 0 40 80; do
  ASB_L2_PERSIST_MB=$MB timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02e/b_$MB.json 2>gpurun_out/r02e/b_$MB.err
  python -c "import json; d=json.load(open('gpurun_out/r02e/b_$MB.json')); print('persist $MB MB', d['ms_per_step'], d['parity'])"
done
bash tools/variant_bench.sh r02e "-DASB_NO_L2_HINTS"
