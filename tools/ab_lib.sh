#!/bin/bash
# Build an experiment variant of the library into paper_1702_08159_b200/_ab/<name>.so
# with extra nvcc flags (e.g. -DMCK_EXP_NOMUFU); select it at run time with
# MCK_LIB_PATH=paper_1702_08159_b200/_ab/<name>.so.
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p paper_1702_08159_b200/_ab
MCK_NVCC_EXTRA="$*" python -c "
import paper_1702_08159_b200.build as b, pathlib, shutil
b.BUILD = pathlib.Path('paper_1702_08159_b200/_ab/build_$name'); b.LIB = pathlib.Path('paper_1702_08159_b200/_ab/$name.so')
print(b.build())"
