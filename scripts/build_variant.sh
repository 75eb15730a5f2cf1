# Build a variant librfxc.so into variants/<name>.so with extra nvcc -D flags
# for one source file:  bash scripts/build_variant.sh NAME FILE.cu "-DFOO=1 ..."
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; defs=$3
B=paper_2511_19493_b200/_build; C=paper_2511_19493_b200/csrc
mkdir -p variants/obj_$name
objs=""
for o in $B/obj/*.o; do
  base=$(basename $o .o)
  if [ "$base.cu" = "$src" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $defs -c $C/$src -o variants/obj_$name/$base.o -Xptxas -v 2> variants/obj_$name/ptxas.txt
    objs="$objs variants/obj_$name/$base.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so $objs -lcudart_static -lrt -lpthread -ldl
echo built variants/$name.so
