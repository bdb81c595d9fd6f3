# builds rowres variants under build/variants (development aid)
set -e
mk() { ATKG_VARIANT_TAG=_$1 ATKG_BUILD_LIB=build/variants/$1.so ATKG_DEFINES="$2" python paper_2506_04165_b200/build.py > /dev/null; }
mkdir -p build/variants
rm -f build/variants/*.so
mk ilp2 "-DATKG_RR_ILP2"
mk nop2 "-DATKG_RR_NOPASS2"
mk nop2ilp2 "-DATKG_RR_NOPASS2 -DATKG_RR_ILP2"
mk nofast "-DATKG_RR_NOFAST"
mk nofastilp2 "-DATKG_RR_NOFAST -DATKG_RR_ILP2"
