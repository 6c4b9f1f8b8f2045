# A/B: the next ticket and an acquire read of its dependency counter issued while the
# current unit's input is in flight (variant eacq: MXB_PIPE_EARLY_ACQ=1)
set -x
P=gpurun_out/eacqab
MXB_LIB=variants/eacq/libmagnex_b200.so timeout 1200 python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py tests/test_full_size.py tests/test_slab.py tests/test_xstage.py -q -x > ${P}_tests_eacq.txt 2>&1
for r in 1 2 3; do
  for V in default eacq; do
    case $V in
      default) unset MXB_LIB ;;
      *) export MXB_LIB=variants/$V/libmagnex_b200.so ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
