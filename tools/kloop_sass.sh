#!/bin/bash
# SASS of the promotion k-loop of one K1 instantiation in a given libtagg build:
# the instructions between the first and last LDTM of the full-tile path, with a summary.
LIB=${1:-paper_2508_16584_b200/libtagg.so}; FN=${2:-_ZN4tagg16tagg_gemm_kernelILi2ELi256ELb0ELb1EEEvNS_6ParamsE}
T=$(mktemp -d); LIB=$(readlink -f $LIB)
(cd $T && cuobjdump -xelf all $LIB >/dev/null 2>&1 && cuobjdump -sass -fun $FN tagg_gemm.sm_100a.cubin > k.sass 2>/dev/null)
grep -E "^\s+/\*[0-9a-f]{4}\*/" $T/k.sass | sed 's@/\* 0x[0-9a-f]* \*/@@' > $T/k.txt
wc -l < $T/k.txt
grep -n "LDTM" $T/k.txt | head -20
rm -rf $T
