# usage: bash scripts/ab_build.sh GITREF NAME [EXTRA]  -- build libskv_b200.so of csrc at GITREF into build_var/libNAME.so (A/B timing)
set -e
ROOT=$(cd $(dirname $0)/.. && pwd)
TMP=$(mktemp -d)
git -C $ROOT archive $1 paper_2403_17312_b200/csrc include | tar -x -C $TMP
make -s -C $TMP/paper_2403_17312_b200/csrc EXTRA="$3" OBJDIR=$TMP/obj OUT=$ROOT/build_var/lib$2.so > /dev/null
rm -rf $TMP
echo built build_var/lib$2.so
