# e2e A/B of the prefaulted final readback array (MXB_PREFAULT=0 disables it)
set -x
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pf_tests.txt 2>&1
for V in 0 1 0 1 0 1; do
  echo "$V $(MXB_PREFAULT=$V python bench.py --steps 20 --warmup 3 --repeats 1 --no-cpu 2>>gpurun_out/pf_bench.err)" >> gpurun_out/pf_bench_all.txt
done
