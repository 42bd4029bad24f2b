# N = 1 bench of every BASELINE config with the current kernels -> gpurun_out/sweep_<cfg>.json
for c in cfg2 cfg3 cfg4_cb_B512 cfg4_cb_B1024 cfg4_cb_B2048 cfg4_sq_B2048 cfg5_B8192 cfg5; do
  timeout 900 python bench.py --config $c --secondary "" --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err
  python -c "import json; d=json.load(open('gpurun_out/sweep_$c.json')); r=d['roofline']['per_kernel']; print('$c', round(d['value'],1), round(d['ms_per_step'],2), 'fwd', round(r['attn_fwd_kernel']['tflops'],1), 'bwd', round(r['attn_bwd_kernel']['tflops'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
