# A/B: unrolled B-multiply kernel-entry loop (MXB_PIPE_KUNROLL 2, 3)
set -x
P=gpurun_out/kuab
MXB_LIB=variants/ku2/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py -q -k "warp or l1024" > ${P}_tests.txt 2>&1
for V in default ku2 ku3 default ku2 ku3 default ku2 ku3; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
