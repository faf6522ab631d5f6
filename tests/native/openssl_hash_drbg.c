/* TEST-ONLY harness (tests/test_oracle_standard_pins.py): drives OpenSSL 3's EVP_RAND "HASH-DRBG"
 * (SHA-256) seeded through the deterministic "TEST-RAND" parent, so the Hash_DRBG oracle
 * (oracle/drbg.py, SP 800-90A §10.1.1; R20) is pinned to an independent implementation of the
 * standard.  Returns 0 on success, a negative step number on failure. */
#include <openssl/evp.h>
#include <openssl/core_names.h>
#include <openssl/params.h>
#include <stdio.h>
#include <string.h>
#include <stdint.h>
int hash_drbg(const unsigned char* entropy, size_t elen, const unsigned char* nonce, size_t nlen,
              const unsigned char* pers, size_t plen, const size_t* req, int nreq, unsigned char* out)
{
  unsigned int strength = 256;
  EVP_RAND *trand = EVP_RAND_fetch(NULL, "TEST-RAND", NULL);
  EVP_RAND_CTX *parent = EVP_RAND_CTX_new(trand, NULL);
  OSSL_PARAM p[4];
  p[0] = OSSL_PARAM_construct_uint(OSSL_RAND_PARAM_STRENGTH, &strength);
  p[1] = OSSL_PARAM_construct_octet_string(OSSL_RAND_PARAM_TEST_ENTROPY, (void*)entropy, elen);
  p[2] = OSSL_PARAM_construct_octet_string(OSSL_RAND_PARAM_TEST_NONCE, (void*)nonce, nlen);
  p[3] = OSSL_PARAM_construct_end();
  if (!EVP_RAND_CTX_set_params(parent, p)) return -1;
  if (!EVP_RAND_instantiate(parent, strength, 0, NULL, 0, NULL)) return -2;
  EVP_RAND *hrand = EVP_RAND_fetch(NULL, "HASH-DRBG", NULL);
  EVP_RAND_CTX *ctx = EVP_RAND_CTX_new(hrand, parent);
  OSSL_PARAM q[2];
  q[0] = OSSL_PARAM_construct_utf8_string(OSSL_DRBG_PARAM_DIGEST, "SHA256", 0);
  q[1] = OSSL_PARAM_construct_end();
  if (!EVP_RAND_CTX_set_params(ctx, q)) return -3;
  if (!EVP_RAND_instantiate(ctx, strength, 0, pers, plen, NULL)) return -4;
  size_t off = 0;
  for (int i = 0; i < nreq; i++) {
    if (!EVP_RAND_generate(ctx, out + off, req[i], strength, 0, NULL, 0)) return -5 - i;
    off += req[i];
  }
  EVP_RAND_CTX_free(ctx); EVP_RAND_free(hrand); EVP_RAND_CTX_free(parent); EVP_RAND_free(trand);
  return 0;
}
