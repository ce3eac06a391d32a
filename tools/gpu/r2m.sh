python -m pytest tests/test_gpu_cli.py -q -m gpu -p no:cacheprovider > gpurun_out/r2m_pytest.log 2>&1
for c in "scanselftest --len 1024 --d 8 --blocks 4,16,64" "errbench --op square --low 1e-6 --high 1e6 --samples 2000 --backing 32" "errbench --op identity --low 1e-10 --high 1e10 --samples 2000 --backing 64" "errbench --op log --samples 400" "errbench --op add --samples 400" "ssm --d 8 --T 512 --rho 1.5 --check" "lyapunov lle --system henon --steps 30000 --method par"; do
echo "=== $c"; python -m paper_2510_03426_b200 $c 2>&1 | grep -v "^[0-9]" | tail -12; echo "rc=$?"
done > gpurun_out/r2m_cli.log 2>&1
