mkdir -p gpurun_out
rm -f gpurun_out/c2_ab2.txt
for v in "GOOM_TC_DEBUG=0" "GOOM_TC_DEBUG=6" "GOOM_TC_DEBUG=7" "GOOM_TC_DEBUG=16"; do env $v timeout 120 python tools/lmme_prof2.py 128 1024 15 >> gpurun_out/c2_ab2.txt 2>&1; echo "  $v" >> gpurun_out/c2_ab2.txt; done
