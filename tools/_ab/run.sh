# dev A/B of two builds of the library on ONE box (box-to-box spread is ~3 %): copy the two
# libbidomain_b200.so builds to tools/_ab/base.bin and tools/_ab/new.bin, then
#   gpurun -- bash tools/_ab/run.sh
for r in 1 2 3; do for v in base new; do cp tools/_ab/$v.bin paper_1711_08708_b200/libbidomain_b200.so; MODES=btile@rpipe timeout 300 python tools/trsv_bench.py 128,128,64 40 2>&1 | grep -E "us per apply" | sed "s/^/$v /"; done; done
