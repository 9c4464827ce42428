# dev sweep: inbox polling x kernel x CTAs/SM on the cfg2 slab (fwd+bwd pair)
for ib in 0 1; do
  BD_BTILE_INBOX=$ib MODES=btile@reg,btile@rsmem%persm5,btile@rsmem%persm6,btile@rsmem%persm8 python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|rel diff" | sed "s/^/inbox=$ib /"
done
