# Same-box A/B of whole-library variants through an unmodified script: runs CMD with the in-tree
# libssmtp.so, then with build/ab/<name>/.../libssmtp.so swapped in (box copy only), twice.
#   bash scripts/so_ab.sh NAME 'python bench.py ...'
NAME=$1; CMD=$2
SO=paper_2602_21144_b200/libssmtp.so
cp $SO /tmp/base_libssmtp.so
for rep in 1 2; do
  cp /tmp/base_libssmtp.so $SO; echo "== base"; eval "$CMD"
  cp build/ab/$NAME/$SO $SO; echo "== $NAME"; eval "$CMD"
done
cp /tmp/base_libssmtp.so $SO
