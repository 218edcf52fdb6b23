# Build libirk.so of a git revision (default HEAD) into lib/variants/libirk_<name>.so for tools/ab.py
set -e
REV=${1:-HEAD}; NAME=${2:-base}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=$(mktemp -d /tmp/irk_wt_XXXX)
git -C "$ROOT" worktree add -q --detach "$WT" "$REV"
(cd "$WT" && python -c "from paper_2511_03655_b200 import build; build.build(force=True)" > /dev/null)
mkdir -p "$ROOT/paper_2511_03655_b200/lib/variants"
cp "$WT/paper_2511_03655_b200/lib/libirk.so" "$ROOT/paper_2511_03655_b200/lib/variants/libirk_$NAME.so"
git -C "$ROOT" worktree remove --force "$WT"
echo "$ROOT/paper_2511_03655_b200/lib/variants/libirk_$NAME.so"
