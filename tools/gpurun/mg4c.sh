for lib in paper_2308_01241_b200/libvxb.so build/variants/libvxb_scan1.so build/variants/libvxb_scan4.so paper_2308_01241_b200/libvxb.so; do
for n in 4 2; do
VXB_LIB=$lib timeout 1200 python bench.py --gpus $n --steps 20 --warmup 3 --no-cpu > gpurun_out/g4c.log 2>&1
echo "$lib n=$n $(grep '^{' gpurun_out/g4c.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step','exchange_arrival_lag_us_per_step']})")"
done; done
