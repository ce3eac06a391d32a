# launch list + full ncu capture of the long-chain engine's level-0 passes (d = 8, 32)
for d in 8 32; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches_d$d.csv python tools/long_prof.py $d > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:long_fold --launch-skip 0 --launch-count 1 -o gpurun_out/r2j_long_R0_d$d python tools/long_prof.py $d > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:long_fold --launch-skip 8 --launch-count 1 -o gpurun_out/r2j_long_S0_d$d python tools/long_prof.py $d > /dev/null 2>&1
done
ls -la gpurun_out/ | grep r2j
