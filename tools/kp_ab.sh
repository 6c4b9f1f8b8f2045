# A/B: first B kernel entry loaded before the spectrum store and barrier (MXB_PIPE_KPRE)
set -x
P=gpurun_out/kpab
MXB_LIB=variants/kpre/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py -q -k "warp or l1024" > ${P}_tests.txt 2>&1
for V in default kpre default kpre default kpre; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
