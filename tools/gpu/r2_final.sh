# round-2 final evidence: GPU suite, smoke, default bench (+ --impl reference), ncu launch list and
# phase captures, config-2 sweep, small-d long chains
mkdir -p gpurun_out
TAG=r2f2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 python tools/config2_lmme_sweep.py > gpurun_out/${TAG}_config2_sweep.json 2> gpurun_out/${TAG}_config2_sweep.err
timeout 900 python tools/small_d_bench.py --ds 8,16,32,64 --reps 3 --cpu-sample 256 --engines long > gpurun_out/${TAG}_small_d_long.jsonl 2> gpurun_out/${TAG}_small_d.err
TAG=${TAG} bash tools/gpu_profile.sh
