# Build the library with extra nvcc flags into paper_2504_14966_b200/_variants/<name>.so (A/B runs:
# tools/gpu_quick.sh times every variant), then restore the default build (forced: the variant's
# objects are newer than the sources).
#   bash tools/build_variant.sh <name> [nvcc flags...]
set -e
name=$1; shift
SLO_EXTRA_NVCC="$*" python -m paper_2504_14966_b200.build --force > /dev/null
mkdir -p paper_2504_14966_b200/_variants
cp paper_2504_14966_b200/libslosched_b200.so paper_2504_14966_b200/_variants/$name.so
python -m paper_2504_14966_b200.build --force > /dev/null
