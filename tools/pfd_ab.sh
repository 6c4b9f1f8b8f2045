# A/B: (1) r2c L2 prefetch distance (MXB_XW_PFD, run time; default 296), (2) pipeline
# L2 prefetch of the A unit's XP row D tickets ahead (variants pfdD: MXB_PIPE_PF_NEXT=1,
# MXB_PIPE_PF_DIST=D)
set -x
P=gpurun_out/pfdab
for V in pfd1024 pfd2048 pfd4096; do
  MXB_LIB=variants/$V/libmagnex_b200.so timeout 600 python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py -q -x -k "warp or l1024 or pipeline" > ${P}_tests_$V.txt 2>&1
done
timeout 900 python -m pytest tests/test_pipe.py tests/test_full_size.py tests/test_gpu_parity.py -q -x > ${P}_tests_default.txt 2>&1
for r in 1 2; do
  for V in x296 x0 x148 x444 pfd1024 pfd2048 pfd4096; do
    case $V in
      x*) unset MXB_LIB; export MXB_XW_PFD=${V#x} ;;
      *) export MXB_LIB=variants/$V/libmagnex_b200.so; unset MXB_XW_PFD ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
