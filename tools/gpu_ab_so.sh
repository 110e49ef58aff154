#!/bin/bash
# A/B of prebuilt library variants ab/<name>/libigabem_b200.so (tools/build_variant.sh):
# each is swapped in, then SCRIPT (default tools/ab_far.py) runs with the variant name
mkdir -p gpurun_out
cp paper_1906_00785_b200/libigabem_b200.so /tmp/lib_tree.so
for v in ${VARIANTS:-$(ls ab)} tree; do
  if [ "$v" = tree ]; then cp /tmp/lib_tree.so paper_1906_00785_b200/libigabem_b200.so; else cp ab/$v/libigabem_b200.so paper_1906_00785_b200/; fi
  timeout 600 python ${SCRIPT:-tools/ab_far.py} $v 2>&1 | tail -3
done
cp /tmp/lib_tree.so paper_1906_00785_b200/libigabem_b200.so
