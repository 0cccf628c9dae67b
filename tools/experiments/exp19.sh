for o in 0 1 2; do BC_SO=build_exp/lib_dbg.so python - << PY
import sys; sys.path.insert(0,'.')
import graphgen as gg, paper_1602_00963_b200 as bcb
g=gg.rmat(20,16,seed=1); S=gg.sample_sources(g,8192,seed=2)
G=bcb.Graph.from_csr(g); G.set_option(bcb.OPT_SOURCE_ORDER,$o)
G.compute(S); st=G.stats()
ds=st['dist_sum']; quads=ds//1000000; pairs=ds%1000000
print("order $o hits",st['fwd_hits'],"lanes",st['dag_edges'],"lanes/hit",st['dag_edges']/st['fwd_hits'],"dsum",ds)
PY
done
