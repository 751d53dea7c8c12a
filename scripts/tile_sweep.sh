# Build tile-size variants + stats build, then time each on the bench workload.
set -x
cd paper_2110_06879_b200/csrc
make -s stats >/dev/null
for T in 8 16 32; do make -s OUT=../libgridadmm_t$T.so OBJ=../build_t$T EXTRA_NVFLAGS=-DGA_TILE=$T >/dev/null; done
cd ../..
