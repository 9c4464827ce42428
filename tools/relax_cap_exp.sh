# relaxed-supernode block cap (BD_SUPER_RELAX_MAX) on config 1
for cap in ${CAPS:-32 64 128 256 1024}; do
  for fr in ${FRACS:-0.85 0.95}; do
    BD_SUPER_RELAX=$fr BD_SUPER_RELAX_MAX=$cap python tools/cfg_run.py --workload cfg1 --steps 25 > gpurun_out/rc_${cap}_${fr}.log 2>&1
  done
done
