mkdir -p gpurun_out
for v in default build/lib_k6b3.so build/lib_k6b3_k7b3.so build/lib_k6b4.so; do
  if [ "$v" = default ]; then unset PF_LIBRARY_PATH; else export PF_LIBRARY_PATH=$PWD/$v; fi
  echo "== $v" >> gpurun_out/ab.log
  timeout 600 python bench.py --warmup 3 --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fwd_fps'], {k:round(v,3) for k,v in d['stage_ms_per_step'].items() if k in ('K6_forward','K7_backward')})" >> gpurun_out/ab.log 2>&1
done
