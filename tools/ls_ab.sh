# A/B: the previous unit's completion signalled mid-unit (MXB_PIPE_LATE_SIGNAL), and
# without the CTA barrier after the staging wait (MXB_PIPE_NOBAR)
set -x
P=gpurun_out/lsab
for V in lsig lsnb; do
  MXB_LIB=variants/$V/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py tests/test_full_size.py -q -k "warp or l1024 or pipeline or steps" > ${P}_tests_$V.txt 2>&1
done
for V in default lsig lsnb default lsig lsnb default lsig lsnb; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
