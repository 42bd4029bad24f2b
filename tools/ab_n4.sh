# per-rank A/B at N (default 4) GPUs: bench variants as lines of extra arguments on stdin,
# optionally prefixed "LIB=<path to libdcpx.so>"; CONFIGS (default "cfg2 cfg3"), two passes
P=29800
n=${N:-4}
mapfile -t variants
for rep in 1 2; do for c in ${CONFIGS:-cfg2 cfg3}; do for v in "${variants[@]}"; do
  P=$((P+1)); lib=""; args="$v"
  if [[ "$v" == LIB=* ]]; then lib="${v%% *}"; lib="${lib#LIB=}"; args="${v#* }"; [ "$args" = "$v" ] && args=""; fi
  if [ "$n" = 1 ]; then
    r=$(DCPX_LIB=$lib python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --secondary= --config $c $args 2>/dev/null | tail -1)
  else
    r=$(DCPX_LIB=$lib python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --secondary= --config $c $args 2>/dev/null | tail -1)
  fi
  echo "$r" >> gpurun_out/ab_n${n}.jsonl
  echo "N=$n $c [$v]: $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline']['per_kernel']; print(round(d['value'],1), round(d['ms_per_step'],3), {k[5:8]: round(v['gpu_ms_per_step'],2) for k,v in pk.items()})")"
done; done; done
