# usage: bash scripts/build_variant.sh <name> "<extra nvcc flags>"  -> build/var_<name>/libdgvv.so
set -e
DGVV_BUILD_DIR=$PWD/build/var_$1 DGVV_EXTRA_FLAGS="$2" python -m paper_2506_14424_b200.build --jobs 16 > /dev/null
echo build/var_$1/libdgvv.so
