# config 1: rows per dense-phase slice (BD_SUPER_DCHUNK)
for dc in ${DCS:-32 64 128}; do
  BD_SUPER_DCHUNK=$dc python tools/cfg_run.py --workload cfg1 --steps 25 > gpurun_out/dc_$dc.log 2>&1
done
