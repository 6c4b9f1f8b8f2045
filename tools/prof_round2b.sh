# Round-2 second measurement pass (after the pipeline / stage / e2e changes):
# GPU tests, smoke, bench, reference arm, slab bench path checks (2 ranks on one
# GPU with gloo: strong 64^3 and the weak-scaling ladder's N=2 point), N=1 weak
# line, the ncu launch list and --set full captures.  Outputs: gpurun_out/r2b_*.
set -x
P=${P:-gpurun_out/r2b}
python -m pytest tests -m gpu -q > ${P}_gpu_all.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.txt 2>&1
python bench.py > ${P}_bench.json 2> ${P}_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > ${P}_bench_reference.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --backend gloo --size 64 --steps 3 --warmup 1 > ${P}_slab_gloo.json 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29534 bench.py --gpus 2 --backend gloo --scaling weak --steps 2 --warmup 1 > ${P}_slab_weak.json 2>&1
python bench.py --scaling weak --steps 5 --warmup 3 --repeats 2 --no-cpu --no-ref-mode > ${P}_weak1.json 2>&1
python bench.py --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu --no-dev --no-ref-mode > ${P}_b2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file ${P}_launches.csv \
    python bench.py --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu --no-dev --no-ref-mode > ${P}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_r2c_w|k_yz_pipe_w|k_c2r_w|k_stage_zt" -c 7 \
    -o ${P}_prof512 python tools/profile_step.py --n 512 --steps 1 > ${P}_ncu2.log 2>&1
python tools/bench_configs.py > ${P}_configs.jsonl 2>${P}_configs.err
ls -la gpurun_out/ | grep r2
