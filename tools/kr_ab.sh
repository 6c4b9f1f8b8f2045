# A/B: B multiply kernel entries -- loaded 1 / 2 iterations ahead into registers
# (krot1, krot2: MXB_PIPE_KROT) or L1-prefetched 1 / 2 ahead (kpf1, kpf2: MXB_PIPE_KPF_L1)
set -x
P=gpurun_out/krab
for V in krot1 krot2 kpf1 kpf2; do
  MXB_LIB=variants/$V/libmagnex_b200.so timeout 600 python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py -q -x -k "warp or l1024 or pipeline" > ${P}_tests_$V.txt 2>&1
done
for r in 1 2; do
  for V in default krot1 krot2 kpf1 kpf2; do
    case $V in
      default) unset MXB_LIB ;;
      *) export MXB_LIB=variants/$V/libmagnex_b200.so ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
