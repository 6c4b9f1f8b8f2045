# A/B: unrolled B-multiply kernel-entry loop (MXB_PIPE_KUNROLL 2, 3) and cached plane-completion observations (MXB_PIPE_SEEN)
set -x
P=gpurun_out/kuab
for V in ku2 seen; do MXB_LIB=variants/$V/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py -q -k "warp or l1024" > ${P}_tests_$V.txt 2>&1; done
for V in default ku2 ku3 seen default ku2 ku3 seen default ku2 ku3 seen; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
