# concurrent pipelines: GPU-side start offset of pipeline i (BC_STAGGER_US x i), S20 8192 sources, 3 pipelines (auto)
for us in 0 1000 2000 3000 4500 0 1000 2000 3000 4500; do
  echo -n "stagger ${us}us S20 auto: "; BC_STAGGER_US=$us BC_SO=build_exp/lib_st.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
for us in 0 2000; do
  echo -n "stagger ${us}us S20 2pipe: "; BC_STAGGER_US=$us BC_SO=build_exp/lib_st.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --streams 2 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
