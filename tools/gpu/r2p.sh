timeout 600 python -m pytest tests/test_gpu_core.py -q -m gpu -p no:cacheprovider -x -k "fused_scales or square_sweep or rectangular or huge" 2>&1 | tail -15
timeout 300 python tools/config2_lmme_sweep.py > gpurun_out/r2p_c2.json 2> gpurun_out/r2p_c2.err
python -c "
import json; d=json.load(open('gpurun_out/r2p_c2.json'))
for r in d['rows']: print(r['d'], round(r['ms'],3), round(r['roofline_frac'],3), r['parity_rel_log'], r['sign_flips'], {k:round(v,3) for k,v in r['kernels_ms'].items()})"
