# builds rowres variants under build/variants (development aid)
set -e
mk() { ATKG_VARIANT_TAG=_$1 ATKG_BUILD_LIB=build/variants/$1.so ATKG_DEFINES="$2" python paper_2506_04165_b200/build.py > /dev/null; }
mkdir -p build/variants
rm -f build/variants/*.so
mk noext "-DATKG_RR_NOEXTRACT"
mk nop2 "-DATKG_RR_NOPASS2"
