# usage: bash tools/build_variants.sh name1:"-DX=1 -DY=2" name2:"..."  -> build_exp/lib_<name>.so
mkdir -p build_exp
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared -Xptxas -v \
    $defs -Iinclude -o build_exp/lib_$name.so paper_1602_00963_b200/csrc/bc_api.cu > build_exp/lib_$name.log 2>&1 &
done
wait
for spec in "$@"; do
  name=${spec%%:*}
  echo "$name: $(grep -A3 'Compiling entry.*lanes_level_kernelILi4Ed' build_exp/lib_$name.log | grep -E 'spill|Used' | tr '\n' ' ')"
done
