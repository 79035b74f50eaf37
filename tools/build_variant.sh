#!/bin/bash
# A/B build of the library with extra defines: tools/build_variant.sh name "-DFOO -DBAR"
# -> build/var_<name>/librtpb.so (load with RTPB_LIB=...).
set -e
make -s -j8 lib OBJDIR=build/var_$1/obj OUT=build/var_$1/librtpb.so EXTRA="$2"
