# A/B: L2 prefetch of the next A unit's XP row (MXB_PIPE_PF_NEXT) in k_yz_pipe_w
set -x
P=gpurun_out/pfab
MXB_LIB=variants/pfn/libmagnex_b200.so python -m pytest tests/test_pipe.py -q -k "warp" > ${P}_tests.txt 2>&1
for V in default pfn default pfn default pfn; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 5 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
unset MXB_LIB
python -m pytest tests/test_gpu_parity.py -q -s -k "newell_builder or built_kernel_field" > ${P}_tol.txt 2>&1
