# build/var_<name>/libpclab_b200.so with extra nvcc flags: tools/build_variant.sh <name> <flags...>
name=$1; shift
mkdir -p build/var_$name
make -s -C paper_2412_07127_b200/csrc -j8 OBJ=$PWD/build/var_$name/obj OUT=$PWD/build/var_$name/libpclab_b200.so NVFLAGS_EXTRA="$*" 2>&1 | grep -v "^$" | tail -3
grep -A3 "bss_trsv_kernelILb0" build/var_$name/obj/bss.ptxas.log | grep -E "registers|spill"
