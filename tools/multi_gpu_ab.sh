# A/B of the copy-kernel unroll (16-byte loads in flight per thread) at N = 4 (per-rank mode)
P=29600
run() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],3), round(r['plan_roofline_frac'],3))"; }
for i in 1 2; do
echo U4; run
echo U8; DCPX_LIB=build/cu8/libdcpx.so run
echo U16; DCPX_LIB=build/cu16/libdcpx.so run
done
for v in "" build/cu8/libdcpx.so build/cu16/libdcpx.so; do DCPX_LIB=$v python tools/nvlink_probe.py cfg3_R4 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['fwd_ms'], d['bwd_ms'], d['gbs_weighted'], d['gbs_large_median'])"; done
