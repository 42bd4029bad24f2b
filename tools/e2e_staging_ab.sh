for rep in 1 2; do for lib in "" build/stage3/libdcpx.so build/stage4/libdcpx.so; do
 r=$(DCPX_LIB=$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline --secondary= 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(d['value'],1), round(e['value'],1), round(e['ms_per_step'],2), round(e['pcie_frac'],3))")
 echo "lib=[$lib] $r"
done; done
