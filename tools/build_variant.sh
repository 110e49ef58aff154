#!/bin/bash
# build a compile-time variant of libigabem_b200.so into ab/<name>/ (A/B on the GPU box);
# only igb_device.o is rebuilt with the extra nvcc flags
name=$1; shift
d=/tmp/abbuild_$name; rm -rf $d; mkdir -p $d/pkg
cp -r include $d/
cp -rp paper_1906_00785_b200/csrc paper_1906_00785_b200/Makefile paper_1906_00785_b200/build $d/pkg/
rm -f $d/pkg/build/igb_device.o
(cd $d/pkg && make -j4 NVFLAGS_EXTRA="$*" > build.log 2>&1) || { echo "build $name failed"; tail $d/pkg/build.log; exit 1; }
mkdir -p ab/$name && cp $d/pkg/libigabem_b200.so ab/$name/ && echo "built $name: $*"
