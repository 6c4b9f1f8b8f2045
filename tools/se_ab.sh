# A/B: previous unit signalled while the next input is in flight (MXB_PIPE_SIGNAL_EARLY), with release reductions

set -x
P=gpurun_out/seab
for V in sige sigerel; do
  MXB_LIB=variants/$V/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py tests/test_full_size.py -q -k "warp or l1024 or pipeline or steps" > ${P}_tests_$V.txt 2>&1
done
for V in default sige sigerel default sige sigerel default sige sigerel; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
