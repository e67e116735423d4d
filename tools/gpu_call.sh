for v in base ringest base ringest; do echo "== $v"; MSV_LIB=_ab/$v.so timeout 600 python tools/_nb1.py; done
