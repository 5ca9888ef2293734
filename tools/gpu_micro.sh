set -x
./tools/micro/chain_latency
python tools/prep_profile.py > gpurun_out/prep_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/prep_plain.log
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"stats_chain|envelope_gw|stats_convert" -c 3 \
  -o gpurun_out/prep_full --force-overwrite python tools/prep_profile.py > gpurun_out/prep_ncu.log 2>&1; echo "ncu rc=$?"
