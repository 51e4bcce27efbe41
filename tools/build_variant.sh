# Build an A/B variant of the package into exp/<name>/paper_2011_08170_b200 (git-ignored; travels
# to the GPU box with gpurun): tools/build_variant.sh <name> "<extra nvcc flags>"
set -e
name=$1; flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
dst=$root/exp/$name/paper_2011_08170_b200
rm -rf "$root/exp/$name"; mkdir -p "$dst"
cp -r "$root/paper_2011_08170_b200/csrc" "$root/paper_2011_08170_b200/Makefile" "$root/paper_2011_08170_b200/__init__.py" \
      "$root/paper_2011_08170_b200/sharded.py" "$dst/"
make -s -j8 -C "$dst" ROOT="$root" NVFLAGS_EXTRA="$flags"
echo "built $dst"
