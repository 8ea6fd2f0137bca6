for r in 1 2 3; do for g in 0 8; do echo "G=$g $(HLF_RASTER=$g python tools/time_kernel.py 3 3 512x512x256 10)"; done; done
for g in 0 8; do echo "m2 G=$g $(HLF_RASTER=$g python tools/time_kernel.py 3 2 512x512x256 10)"; echo "m1 G=$g $(HLF_RASTER=$g python tools/time_kernel.py 3 1 512x512x256 10)"; done
