#!/bin/bash
# Build a variant of libllmpilot.so with extra nvcc flags for fit.cu into _abv/NAME (a package copy
# that tools/ab_fit.py loads with AB_ROOT=_abv/NAME):  bash tools/build_variant.sh NAME "-DFOO=1 ..." [GITREV]
# (GITREV: take csrc/ from that commit instead of the working tree)
set -e
NAME=$1; FL=$2
R=$(cd "$(dirname "$0")/.." && pwd)
D=$R/_abv/$NAME
mkdir -p $D/paper_2410_02425_b200/build
cp $R/paper_2410_02425_b200/__init__.py $D/paper_2410_02425_b200/
ln -sfn $R/synth $D/synth
ln -sfn $R/oracle $D/oracle
SRC=$R/paper_2410_02425_b200/csrc
if [ -n "$3" ]; then
  SRC=$D/paper_2410_02425_b200/csrc; rm -rf $SRC
  (cd $R && git archive $3 paper_2410_02425_b200/csrc | tar -x -C $D)
  ln -sfn $R/include $D/include
fi
NV=/usr/local/cuda/bin/nvcc
# every translation unit with the variant's flags (in parallel)
for CU in $SRC/*.cu; do
  B=$(basename $CU .cu)
  $NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -I $R/include $FL \
    -c $CU -o $D/paper_2410_02425_b200/build/$B.o &
done
wait
$NV -gencode arch=compute_100a,code=sm_100a -shared -o $D/paper_2410_02425_b200/libllmpilot.so $D/paper_2410_02425_b200/build/*.o -ldl
echo built $D
