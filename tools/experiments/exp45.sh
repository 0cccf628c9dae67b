# threads per CTA of slices_lowdeg_sm_kernel in BFS order (2 CTAs per SM; grid 512x512, 8192 sources)
for v in t384 t448 t512 t576 t640 t512; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done
