# rebuild libgm_b200.so and the ahead-of-time region cubins (after any skeleton/codegen change)
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2509_16248_b200/csrc > /dev/null
rm -rf paper_2509_16248_b200/_kcache
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "rebuilt: $(ls paper_2509_16248_b200/_kcache | wc -l) cubins"
