#include "qtrain_oracle.h"
int qto_version(void) { return 1; }
