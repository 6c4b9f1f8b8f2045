# A/B: kernel-row loads with the evict_first hint (MXB_PIPE_HINT_K) -- same kernel
# time, less DRAM traffic, so more clock headroom under the power cap
set -x
P=gpurun_out/hkab
MXB_LIB=variants/kph1k/libmagnex_b200.so python -m pytest tests/test_pipe.py -q -k "warp" > ${P}_tests.txt 2>&1
for V in default kph1k default kph1k default kph1k; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
