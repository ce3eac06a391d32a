for d in 128 256 512; do python tools/lmme_prof2.py $d 1024 5; done
timeout 600 python -m pytest tests/test_gpu_core.py tests/test_gpu_scan.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
