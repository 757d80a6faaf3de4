# Build libilans_b200.so from the csrc of a git revision (or the work tree)
# into ab_libs/<name>.so, for tools/ab_bench.sh.
# usage: bash tools/ab_build.sh <rev|WORKTREE> <name>
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p $tmp/pkg/csrc $tmp/include $root/ab_libs
if [ "$rev" = WORKTREE ]; then
  cp $root/paper_1402_3392_b200/csrc/* $tmp/pkg/csrc/; cp $root/include/* $tmp/include/
else
  git -C $root archive $rev paper_1402_3392_b200/csrc include | tar -x -C $tmp
  mv $tmp/paper_1402_3392_b200/csrc/* $tmp/pkg/csrc/
fi
cd $tmp/pkg/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  --expt-relaxed-constexpr -I $tmp/include -shared -o $root/ab_libs/$name.so \
  capi.cu table.cu encode.cu decode.cu byte8.cu variant.cu synth.cu mux.cu
rm -rf $tmp
echo built ab_libs/$name.so
